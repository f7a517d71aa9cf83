# launch list of a short c1 (or $1) bench: per-kernel totals
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CFG=${1:-c1}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_l.log 2>&1
echo "ncu rc=$?"
python tools/launch_summary.py gpurun_out/launches_$CFG.csv | head -20
