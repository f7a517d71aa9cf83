cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -30
CMD="python bench.py --pairs 128 --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_screen -s 5 -c 1 -o gpurun_out/prof_screen $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
tail -1 gpurun_out/plain.log
