#!/bin/bash
# A/B of the library builds in build_variants/: tree phase and total (developer tool).
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset EMST_LIB_PATH; else export EMST_LIB_PATH=$PWD/$lib; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ab.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
print('$lib', round(d['value'],1), 'ms', round(d['ms_per_step'],2), d['phase_ms'])" || tail -3 gpurun_out/ab.log
done
