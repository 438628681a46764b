#!/bin/bash
# e2e A/B (developer tool): SPECS as in ab_env_lib.sh; prints the device ms and the e2e ms (pageable
# numpy through boruvka_emst) of each spec, REPS interleaved rounds per config.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS:-blobs3d_37m}; do
for rep in $(seq ${REPS:-2}); do
for spec in $SPECS; do
  IFS='|' read -r label envs lib <<< "$spec"
  if [ "$lib" = default ] || [ -z "$lib" ]; then libenv=""; else libenv="EMST_LIB_PATH=$PWD/$lib"; fi
  env $libenv ${envs//,/ } timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$cfg', '$label', 'dev', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'ok', d['e2e']['parity_ok'])" || tail -3 gpurun_out/ab.log
done
done
done
