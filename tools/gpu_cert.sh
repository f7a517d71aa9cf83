cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
python tools/trace_search.py --config c1 2>&1 | grep -v Warn | tail -12
rm -f gpurun_out/variants_summary.txt
bash tools/gpu_variants.sh c1 > /dev/null 2>&1; cat gpurun_out/variants_summary.txt
LTSG_NO_CERT=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-allpairs 2>&1 | tail -1 | cut -c1-200
