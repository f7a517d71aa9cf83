# Round profile, part A: default bench, reference arm, other configs, then the launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_default.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-300
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-allpairs > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-200
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
