#!/bin/bash
# A/B (developer tool): "label|ENV=.. ENV2=..|lib" specs, REPS interleaved rounds, per config.
# usage: SPECS="new||default base||build_variants/base.so norunner|EMST_RUNNER=0|default" CFGS="blobs3d_37m" bash tools/ab_env_lib.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS:-blobs3d_37m}; do
for rep in $(seq ${REPS:-2}); do
for spec in $SPECS; do
  IFS='|' read -r label envs lib <<< "$spec"
  if [ "$lib" = default ] || [ -z "$lib" ]; then libenv=""; else libenv="EMST_LIB_PATH=$PWD/$lib"; fi
  env $libenv ${envs//,/ } timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --config $cfg > gpurun_out/ab.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$cfg', '$label', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), 'ok', d['parity']['ok'], [round(r['traverse_ms'],2) for r in d['rounds']][:6], {k: round(v,2) for k,v in d['phase_ms'].items() if k in ('tree','upper_bounds','reduce_labels','merge')})" || tail -3 gpurun_out/ab.log
done
done
done
