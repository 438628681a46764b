# full ncu captures of the round-1 and round-2 traversal of one 37M solve (developer tool)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${CFG:-blobs3d_37m}
for R in ${ROUNDS:-1 2}; do
  ncu --set full --clock-control none --import-source on -k regex:k_traverse --launch-skip $((R - 1)) --launch-count 1 \
      -o gpurun_out/trav_r${R}_$CFG -f python bench.py --profile --config $CFG > gpurun_out/ncu_trav_r$R.log 2>&1
  echo "round $R exit $?"
done
