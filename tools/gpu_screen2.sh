cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/variants_summary.txt
bash tools/gpu_variants.sh c1 > /dev/null 2>&1; cat gpurun_out/variants_summary.txt
