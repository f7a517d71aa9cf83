# Round-end profile set: bench lines (c1 headline, reference arm, c2..c5, c1 exhaustive),
# the c1 launch list, ncu --set full of k_screen_static (c1) and k_screen (c4).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
for c in c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-allpairs > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
done
timeout 900 python bench.py --exhaustive --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_exh.log 2>&1; echo "exh rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
CMD="python bench.py --config c1 --steps 1 --warmup 3 --no-cpu --no-allpairs"
ncu --set full --clock-control none --import-source on -k "regex:^k_screen_static$" -c 16 -f -o gpurun_out/prof_static $CMD > gpurun_out/ncu_static.log 2>&1
echo "ncu static rc=$?"
CMD="python bench.py --config c4 --pairs 512 --steps 1 --warmup 3 --no-cpu --no-allpairs"
ncu --set full --clock-control none --import-source on -k "regex:^k_screen$" -c 7 -f -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu c4 rc=$?"
