cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --pairs 128 --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
echo "rc=$?"
tail -2 gpurun_out/plain.log
