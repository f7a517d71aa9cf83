# GPU parity suite + smoke, then per-config A/B of the library variants (tools/gpu_variants2.sh)
cd $GRAFT_REPO_ROOT
bash tools/gpu_tests.sh
CFGS="${CFGS:-c4 c5}" STEPS=${STEPS:-5} bash tools/gpu_variants2.sh
