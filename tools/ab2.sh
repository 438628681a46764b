#!/bin/bash
# A/B environment variants of the default library (developer tool)
run() {
  timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$*', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), d['phase_ms']['find_edges'])" || tail -3 gpurun_out/ab.log
}
run X=1
for k in 2 3 4 6; do run EMST_PACKET_FROM=$k; done
for lib in build_variants/*.so; do run EMST_LIB_PATH=$PWD/$lib; done
