#!/bin/bash
# A/B environment settings of the default library on one config (developer tool): CFG=... bash tools/ab_env_cfg.sh "A=1" "A=2"
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config ${CFG:-blobs3d_37m} > gpurun_out/ab.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('${CFG:-blobs3d_37m} $envs', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'tree', d['phase_ms']['tree'], 'trav', round(d['roofline']['ms_per_step'],2), [round(r['traverse_ms'],2) for r in d['rounds']])" || tail -3 gpurun_out/ab.log
done
