for lib in default build_variants/*.so; do
  if [ "$lib" = default ]; then unset EMST_LIB_PATH; else export EMST_LIB_PATH=$PWD/$lib; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_onesweep --csv --log-file gpurun_out/sort_$(basename $lib .so).csv python bench.py --profile --config blobs3d_37m > /dev/null 2>&1
done
REPS=1 bash tools/ab.sh
