cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_tree_api.py tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q --timeout 600 > gpurun_out/pytest2.log 2>&1; echo pytest=$?
for s in 1 0; do EMST_STAGE=$s timeout 300 python tools/e2e_breakdown.py >> gpurun_out/e2e.log 2>&1; done
nproc >> gpurun_out/e2e.log
tail -5 gpurun_out/pytest2.log
cat gpurun_out/e2e.log
