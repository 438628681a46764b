cd $GRAFT_REPO_ROOT
KERNELS="k_onesweep:3 k_onesweep:10" bash tools/ncu_kernels.sh
SAN_N=4000 bash tools/r02_sanitize.sh
