cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
CMD="python bench.py --config c1 --steps 1 --warmup 3 --no-cpu --no-allpairs"
ncu --set full --clock-control none --import-source on -k "regex:^k_screen_static$" -c 16 -f -o gpurun_out/prof_static $CMD > gpurun_out/ncu_static.log 2>&1
echo "ncu static rc=$?"
