#!/bin/bash
run() {
  timeout 300 env "$@" python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${CFG:+--config $CFG} > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$*', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['phase_ms'])
print([ (r['traverse_ms'], r['node_visits'], r['found']) for r in d['rounds']])" || tail -3 gpurun_out/ab.log
}
run EMST_TWO_PASS=1
run EMST_TWO_PASS=0
run EMST_TWO_PASS=1 BENCH_CFG=1
