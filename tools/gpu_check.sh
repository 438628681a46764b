cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench1=$?
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --config normal3d_10m > gpurun_out/bench2.log 2>&1; echo bench2=$?
tail -3 gpurun_out/pytest.log
