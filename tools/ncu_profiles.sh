#!/bin/bash
# The ncu evidence committed under profiles/ (developer tool; one GPU, never under torchrun):
#   launches_<cfg>.csv      every kernel of one solve, gpu__time_duration (serialised, cold caches)
#   trav_dram_<cfg>.csv     DRAM bytes + duration of every traversal launch of one solve
#   trav_r2_<cfg>.ncu-rep   --set full of the round-2 traversal launch (the most expensive round)
mkdir -p gpurun_out
CFG=${CFG:-blobs3d_37m}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv \
    python bench.py --profile --config $CFG > /dev/null 2>&1; echo "launches $?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_traverse \
    --csv --log-file gpurun_out/trav_dram_$CFG.csv python bench.py --profile --config $CFG > /dev/null 2>&1; echo "dram $?"
ncu --set full --clock-control none --import-source on -k regex:k_traverse --launch-skip 1 --launch-count 1 \
    -o gpurun_out/trav_r2_$CFG -f python bench.py --profile --config $CFG > /dev/null 2>&1; echo "full $?"
