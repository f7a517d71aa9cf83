cd $GRAFT_REPO_ROOT
bash tools/gpu_tests.sh
CFGS="c1 c4 c5" STEPS=5 bash tools/gpu_variants2.sh
