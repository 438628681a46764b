#!/bin/bash
# Full-set ncu captures of selected kernels of one bench step (developer tool).
# usage: KERNELS="name:skip name:skip ..." bash tools/ncu_kernels.sh
mkdir -p gpurun_out
CFG=${CFG:-blobs3d_37m}
for spec in ${KERNELS:-k_onesweep:0}; do
  k=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k --launch-skip $skip \
      --launch-count 1 -o gpurun_out/k_${k}_$skip -f python bench.py --profile --config $CFG > gpurun_out/ncu_$k.log 2>&1
  echo "$k:$skip exit $?"
done
