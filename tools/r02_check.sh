#!/bin/bash
# Round-2 GPU evidence (developer tool): tests, smoke, bench lines; everything lands in gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench1=$?
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2.log 2>&1; echo bench2=$?
tail -5 gpurun_out/pytest.log
tail -1 gpurun_out/bench1.log | cut -c1-600
