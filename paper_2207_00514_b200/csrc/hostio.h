// hostio.h -- host <-> device transfers of the host-pointer entry (emst_boruvka
// without EMST_POINTS_ON_DEVICE / EMST_OUTPUT_ON_DEVICE).
//
// A caller of the reference API hands over a plain (pageable) numpy array and
// gets numpy arrays back.  cudaMemcpy from pageable memory is staged by the
// driver on one thread; here the host side is a pipeline instead:
//
//   H2D  the points are cut into chunks; host threads copy chunk i into a
//        page-locked ring slot while the copy engine moves chunk i-1 to HBM.
//   D2H  the edges leave the GPU as packed (u << 32 | v) u64 -- 8 bytes per
//        edge instead of the reference's two int64 -- and host threads widen
//        chunk i into the caller's int64 (n-1, 2) rows while chunk i+1 is in
//        flight; the f64 weights go straight into the caller's buffer when it
//        is page-locked, else through the ring as well.
//
// PCIe volume per 37M-point solve: 444 MB in, 592 MB out (was 888 MB out).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif

namespace emst_host {

// Fixed worker pool; run(parts, fn) calls fn(0..parts-1) on the workers and the
// calling thread and returns when all parts are done.
class ThreadPool {
 public:
  explicit ThreadPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size() + 1; }

  void run(int parts, const std::function<void(int)>& fn) {
    if (parts <= 0) return;
    if (parts == 1 || th_.empty()) {
      for (int p = 0; p < parts; ++p) fn(p);
      return;
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &fn;
      parts_.store(parts);
      next_.store(0);
      pending_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      const int p = next_.fetch_add(1);
      if (p >= parts_) return;
      (*job_)(p);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  std::atomic<int> parts_{0};
  int pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// packed (u << 32 | v) -> int64 (u, v) rows.  Streaming (non-temporal) stores: the rows are written
// once and not read back here, so skipping the read-for-ownership of every output line saves a third
// of the host memory traffic (measured on the B200 box: 37M edges back in 18.3 -> 11.6 ms).
inline void widen_pairs(const unsigned long long* uv, size_t cnt, int64_t* out) {
  size_t i = 0;
#if defined(__SSE2__)
  if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    for (; i < cnt; ++i) {
      const unsigned long long x = uv[i];
      _mm_stream_si128(reinterpret_cast<__m128i*>(out + 2 * i),
                       _mm_set_epi64x((long long)(x & 0xffffffffull), (long long)(x >> 32)));
    }
    _mm_sfence();
    return;
  }
#endif
  for (; i < cnt; ++i) {
    out[2 * i] = (int64_t)(uv[i] >> 32);
    out[2 * i + 1] = (int64_t)(uv[i] & 0xffffffffull);
  }
}

inline bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// The staging ring and its pool, one per context.
struct Stager {
  static constexpr int kMaxSlots = 16;
  int kSlots = 4;                  // (EMST_STAGE_SLOTS)
  size_t kSlotBytes = 16u << 20;   // (EMST_STAGE_MB)
  ThreadPool* pool = nullptr;
  unsigned char* slot[kMaxSlots] = {};
  cudaEvent_t ev[kMaxSlots] = {};
  bool ready = false;

  cudaError_t init() {
    if (ready) return cudaSuccess;
    unsigned hw = std::thread::hardware_concurrency();
    int threads = (int)std::min<unsigned>(hw ? hw : 4, 16u);
    if (const char* t = getenv("EMST_STAGE_THREADS")) threads = std::max(1, atoi(t));
    if (const char* t = getenv("EMST_STAGE_MB")) kSlotBytes = (size_t)std::max(1, atoi(t)) << 20;
    if (const char* t = getenv("EMST_STAGE_SLOTS")) kSlots = std::min(kMaxSlots, std::max(2, atoi(t)));
    int workers = threads - 1;
    pool = new ThreadPool(std::max(workers, 0));
    for (int i = 0; i < kSlots; ++i) {
      cudaError_t e = cudaMallocHost(&slot[i], kSlotBytes);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    ready = true;
    return cudaSuccess;
  }
  void release() {
    for (int i = 0; i < kMaxSlots; ++i) {
      if (slot[i]) cudaFreeHost(slot[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      slot[i] = nullptr;
      ev[i] = nullptr;
    }
    delete pool;
    pool = nullptr;
    ready = false;
  }

  // memcpy on all pool threads, cut at 4 KB boundaries
  void par_copy(void* dst, const void* src, size_t bytes) {
    const int parts = (int)std::min<size_t>((size_t)pool->size(), std::max<size_t>(1, bytes >> 20));
    const size_t per = ((bytes + parts - 1) / parts + 4095) & ~(size_t)4095;
    pool->run(parts, [&](int p) {
      const size_t a = (size_t)p * per, b = std::min(bytes, a + per);
      if (a < b) memcpy((char*)dst + a, (const char*)src + a, b - a);
    });
  }

  // pageable host -> device, queued on `s`; returns once every byte has left the caller's buffer
  cudaError_t h2d(void* dev, const void* host, size_t bytes, cudaStream_t s) {
    const size_t chunks = (bytes + kSlotBytes - 1) / kSlotBytes;
    for (size_t i = 0; i < chunks; ++i) {
      const int k = (int)(i % kSlots);
      if (i >= (size_t)kSlots) {
        cudaError_t e = cudaEventSynchronize(ev[k]);   // that slot's previous chunk has been sent
        if (e != cudaSuccess) return e;
      }
      const size_t off = i * kSlotBytes, len = std::min(kSlotBytes, bytes - off);
      par_copy(slot[k], (const char*)host + off, len);
      cudaError_t e = cudaMemcpyAsync((char*)dev + off, slot[k], len, cudaMemcpyHostToDevice, s);
      if (e != cudaSuccess) return e;
      e = cudaEventRecord(ev[k], s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;   // (later uses of the slots are ordered behind these copies on `s`)
  }

  // One device -> host stream: `unit` bytes per element on the device, `put(dst_index, slot_ptr, count)`
  // turns `count` staged elements into the caller's layout (widening or copying).
  struct Out {
    const void* dev;
    size_t count, unit;
    std::function<void(size_t, const unsigned char*, size_t)> put;
    const cudaEvent_t* ready = nullptr;   // optional: ready[e / ready_per] is recorded once element e exists
    size_t ready_per = 0;
  };

  // device -> host through the ring, the streams' chunks back to back in one pipeline (the copy
  // engine does not drain between two outputs)
  cudaError_t d2h(const std::vector<Out>& outs, cudaStream_t s) {
    struct Chunk { const Out* o; size_t a, len; };
    std::vector<Chunk> ch;
    for (const Out& o : outs) {
      const size_t per = kSlotBytes / o.unit;
      for (size_t a = 0; a < o.count; a += per) ch.push_back({&o, a, std::min(per, o.count - a)});
    }
    auto issue = [&](size_t i) -> cudaError_t {
      const int k = (int)(i % kSlots);
      const Chunk& c = ch[i];
      if (c.o->ready) {   // wait for the producer of the chunk's last element
        cudaError_t e = cudaStreamWaitEvent(s, c.o->ready[(c.a + c.len - 1) / c.o->ready_per], 0);
        if (e != cudaSuccess) return e;
      }
      cudaError_t e = cudaMemcpyAsync(slot[k], (const char*)c.o->dev + c.a * c.o->unit, c.len * c.o->unit,
                                      cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) return e;
      return cudaEventRecord(ev[k], s);
    };
    for (size_t i = 0; i < ch.size() && i < (size_t)kSlots; ++i) {
      cudaError_t e = issue(i);
      if (e != cudaSuccess) return e;
    }
    for (size_t i = 0; i < ch.size(); ++i) {
      const int k = (int)(i % kSlots);
      cudaError_t e = cudaEventSynchronize(ev[k]);
      if (e != cudaSuccess) return e;
      const Chunk& c = ch[i];
      const int parts = (int)std::min<size_t>((size_t)pool->size(), std::max<size_t>(1, c.len >> 17));
      const size_t step = (c.len + parts - 1) / parts;
      pool->run(parts, [&](int p) {
        const size_t b = (size_t)p * step, d = std::min(c.len, b + step);
        if (b < d) c.o->put(c.a + b, slot[k] + b * c.o->unit, d - b);
      });
      if (i + kSlots < ch.size()) {
        e = issue(i + kSlots);
        if (e != cudaSuccess) return e;
      }
    }
    return cudaSuccess;
  }
};

}  // namespace emst_host
