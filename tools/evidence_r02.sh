#!/bin/bash
# Round-2 evidence on one GPU (developer tool): bench lines (ours on every config, the reference arm on
# the headline), ncu launch lists, traversal DRAM per launch and a --set full capture of the round-2
# traversal.  Everything lands in gpurun_out/; tools/make_profile.py r02 composes profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench default $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "reference $?"
for cfg in blobs2d_24m uniform2d_10m normal3d_10m; do
  timeout 400 python bench.py --steps 5 --warmup 3 --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  echo "bench $cfg $?"
done
for cfg in blobs3d_37m blobs2d_24m; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
      python bench.py --profile --config $cfg > /dev/null 2>&1; echo "launches $cfg $?"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_traverse \
      --csv --log-file gpurun_out/trav_dram_$cfg.csv python bench.py --profile --config $cfg > /dev/null 2>&1; echo "dram $cfg $?"
done
ncu --set full --clock-control none --import-source on -k regex:k_traverse --launch-skip 1 --launch-count 1 \
    -o gpurun_out/trav_r2_blobs3d_37m -f python bench.py --profile --config blobs3d_37m > /dev/null 2>&1; echo "full $?"
du -sh gpurun_out
