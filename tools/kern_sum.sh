# per-kernel summed ncu time for the default build and build_variants/*.so (developer tool)
# usage: KREGEX=k_node_labels bash tools/kern_sum.sh
cd $GRAFT_REPO_ROOT
for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset EMST_LIB_PATH; else export EMST_LIB_PATH=$PWD/$lib; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${KREGEX} --csv \
      --log-file gpurun_out/ks.csv python bench.py --profile --config ${CFG:-blobs3d_37m} > /dev/null 2>&1
  python - "$lib" <<'PY'
import csv, sys
rows = list(csv.reader(open('gpurun_out/ks.csv'))); h = None; t = []
for r in rows:
    if 'Kernel Name' in r: h = r; continue
    if h and len(r) == len(h): t.append(float(r[h.index('Metric Value')]) / 1e3)
print(sys.argv[1], len(t), 'launches', round(sum(t) / 1e3, 3), 'ms', [round(x) for x in t])
PY
done
