cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo bench1=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_blobs3d_37m.csv \
    python bench.py --profile --config blobs3d_37m > /dev/null 2>&1; echo launches=$?
EMST_TRACE=1 EMST_LIB_PATH=$PWD/build_variants/visit_hist.so timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/visit_hist.log 2>&1; echo vh=$?
grep "visits" gpurun_out/visit_hist.log | tail -4
