#!/bin/bash
# Full-set ncu captures of selected kernels of one bench step, exported to small CSVs on the box
# (details page + per-line source counters); the .ncu-rep files are kept only if KEEP=1.
# usage: KERNELS="name:skip ..." CFG=blobs3d_37m bash tools/ncu_export.sh
mkdir -p gpurun_out
CFG=${CFG:-blobs3d_37m}
for spec in ${KERNELS:-k_onesweep:0}; do
  k=${spec%%:*}; skip=${spec##*:}
  rep=gpurun_out/x_${k}_$skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:$k --launch-skip $skip \
      --launch-count 1 -o $rep -f python bench.py --profile --config $CFG > /dev/null 2>&1
  echo "$k:$skip exit $?"
  ncu -i $rep.ncu-rep --page details --csv > ${rep}_details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source cuda,sass > ${rep}_source.csv 2>/dev/null
  gzip -f ${rep}_source.csv
  [ "$KEEP" = 1 ] || rm -f $rep.ncu-rep
done
