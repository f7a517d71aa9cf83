cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --only --config c4 --steps 5 --warmup 3 --no-cpu --no-allpairs > gpurun_out/c4_a.log 2>&1; echo "a rc=$?"
python tools/bench_table.py gpurun_out/c4_a.log | sed -n 2p
LTSG_NO_POSES=1 timeout 900 python bench.py --only --config c4 --steps 5 --warmup 3 --no-cpu --no-allpairs > gpurun_out/c4_b.log 2>&1; echo "b rc=$?"
python tools/bench_table.py gpurun_out/c4_b.log | sed -n 2p
timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -k regex:^k_mscreen\$ -s 5 -c 1 -f -o gpurun_out/prof_mscreen2 python tools/prof_search.py --config c4 --pairs 2048 > gpurun_out/ncu_ms2.log 2>&1
echo "ncu rc=$?"
