#!/bin/bash
# A/B one kernel's summed ncu time (and the bench) across the library builds in build_variants/ (developer tool).
# usage: KREGEX=k_node_labels bash tools/kern_ab.sh
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset EMST_LIB_PATH; else export EMST_LIB_PATH=$PWD/$lib; fi
  name=$(basename $lib .so)
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX} --csv \
      --log-file gpurun_out/kab_$name.csv python bench.py --profile --config ${CFG:-blobs3d_37m} > /dev/null 2>&1
  python - gpurun_out/kab_$name.csv <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = None; tot = 0.0; n = 0
for r in rows:
    if 'Kernel Name' in r: h = r; continue
    if h and len(r) == len(h): tot += float(r[h.index('Metric Value')]); n += 1
print(sys.argv[1], n, 'launches', round(tot / 1e6, 3), 'ms')
PY
done
REPS=${REPS:-1} bash tools/ab.sh
