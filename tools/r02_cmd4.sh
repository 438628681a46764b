# prefilter A/B + full ncu captures of the late-round scan / labelling / prefilter (developer tool)
cd $GRAFT_REPO_ROOT
SPECS="base||build_variants/base.so new||default" CFGS="blobs3d_37m blobs2d_24m" REPS=2 bash tools/ab_env_lib.sh
KERNELS="RoundScanOp:5 k_node_labels_front:5 k_prefilter:4" bash tools/ncu_export.sh
