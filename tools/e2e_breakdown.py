"""Where the end-to-end call spends its time (developer tool)."""
import time, ctypes
import numpy as np, torch
import paper_2207_00514_b200 as E
from paper_2207_00514_b200 import _lib

pts = E.generate(E.DatasetSpec("blobs", 37_000_000, 3, seed=0))
pinned = torch.from_numpy(pts).pin_memory().numpy()
ctx = E.Context(0)
for it in range(3):
    t0 = time.perf_counter()
    res = E.boruvka_emst(pinned, context=ctx)
    t1 = time.perf_counter()
    s = float(np.sum(res.weights))
    t2 = time.perf_counter()
    print(f"call {1e3*(t1-t0):.1f} ms  np.sum {1e3*(t2-t1):.1f} ms  device total {1e3*res.phase_timings['mst']+1e3*res.phase_timings['tree']:.1f} ms")
ne = len(pts) - 1
e = torch.empty((ne, 2), dtype=torch.int64, pin_memory=True).numpy()
w = torch.empty((ne,), dtype=torch.float64, pin_memory=True).numpy()
st = _lib.Stats(); err = _lib.err_buf()
for it in range(3):
    t0 = time.perf_counter()
    rc = _lib.load().emst_boruvka(ctx.handle, pinned.ctypes.data, len(pts), 3, _lib.SUBTREE_SKIP | _lib.UPPER_BOUNDS,
                                  e.ctypes.data, w.ctypes.data, ctypes.byref(st), err, len(err))
    t1 = time.perf_counter()
    print(f"raw C call {1e3*(t1-t0):.1f} ms (phase total {st.phase_ms[7]:.1f} ms, h2d {st.h2d_bytes/1e6:.0f} MB d2h {st.d2h_bytes/1e6:.0f} MB)")
