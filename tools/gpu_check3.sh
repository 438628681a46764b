cd $GRAFT_REPO_ROOT
for cfg in "1 1 16" "1 0 16" "1 1 8"; do set -- $cfg
  echo "== stage=1 packed=$2 threads=$3" >> gpurun_out/e2e3.log
  EMST_STAGE=$1 EMST_PACKED=$2 EMST_STAGE_THREADS=$3 timeout 300 python tools/e2e_breakdown.py 2>&1 | tail -2 >> gpurun_out/e2e3.log
done
cat gpurun_out/e2e3.log
