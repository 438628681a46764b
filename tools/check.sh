#!/bin/bash
# GPU check (developer tool): parity tests, then the headline bench and the per-round traversal profile.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
for cfg in ${CFGS:-blobs3d_37m}; do
  timeout 400 python bench.py --steps 5 --warmup 3 --config $cfg ${BENCH_ARGS} > gpurun_out/bench_$cfg.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bench_$cfg.log').read().strip().splitlines()[-1])
print('$cfg', round(d['value'],1), 'ms', round(d['ms_per_step'],2), 'trav', round(d['roofline']['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), d['phase_ms'])
print([ (round(r['traverse_ms'],2), r['node_visits'], r['found'], r.get('skipped')) for r in d.get('rounds',[])])" || tail -5 gpurun_out/bench_$cfg.log
done
