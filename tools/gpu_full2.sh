# full default bench (all workloads incl. broad phase + contact consumers), reference arm, c1 launch list, ncu of k_mscreen
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1700 python bench.py ) > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_full.log
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu --only"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -k regex:^k_mscreen\$ -s 5 -c 1 -f -o gpurun_out/prof_k_mscreen python tools/prof_search.py --config c4 --pairs 2048 > gpurun_out/ncu_k_mscreen.log 2>&1
echo "ncu mscreen rc=$?"
