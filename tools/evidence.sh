#!/bin/bash
# Round evidence on one GPU (developer tool): tests, smoke, bench lines (ours + reference arm), ncu launch
# lists, traversal DRAM traffic and a --set full capture of the round-2 traversal.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1
for cfg in blobs2d_24m uniform2d_10m normal3d_10m; do
  timeout 400 python bench.py --steps 5 --warmup 3 --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
done
bash tools/ncu_profiles.sh
CFG=blobs2d_24m bash tools/ncu_step.sh
# mutual reachability at the headline size (k_pts 4 and 16)
for k in 4 16; do PYTHONPATH=$PWD timeout 300 python tools/mrd_timing.py blobs3d_37m $k > gpurun_out/mrd_k$k.log 2>&1; done
