#!/bin/bash
# ncu evidence for one bench step (developer tool):
#   1. launch list: per-kernel durations of one full solve (serialised, cold-ish caches)
#   2. a full-set capture of the traversal kernel in round $TRAV_ROUND (default 2)
mkdir -p gpurun_out
CFG=${CFG:-blobs3d_37m}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python bench.py --profile --config $CFG > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
if [ -n "$FULL" ]; then
  R=${TRAV_ROUND:-2}
  ncu --set full --clock-control none --import-source on -k regex:k_traverse --launch-skip $((R - 1)) --launch-count 1 \
      -o gpurun_out/trav_r${R}_$CFG -f python bench.py --profile --config $CFG > gpurun_out/ncu_full.log 2>&1
  echo "full exit $?"
fi
