#!/bin/bash
# A/B environment settings of the default library (developer tool)
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$envs', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), [round(r['traverse_ms'],2) for r in d['rounds']])" || tail -3 gpurun_out/ab.log
done
