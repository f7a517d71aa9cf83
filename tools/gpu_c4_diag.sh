# c4 moving-path diagnosis: per-generation trace (2048 pairs), ncu of k_mscreen / k_mexact (largest generation)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/trace_search.py --config c4 --pairs 2048 > gpurun_out/trace_c4.log 2>&1; echo "trace rc=$?"
grep "ltsg trace" gpurun_out/trace_c4.log | tail -40
for k in k_mscreen k_mexact; do
timeout 900 ncu --nvtx --nvtx-include "prof/" --set full --clock-control none --import-source on \
    -k regex:^$k\$ -s 5 -c 1 -f -o gpurun_out/prof_$k python tools/prof_search.py --config c4 --pairs 2048 > gpurun_out/ncu_$k.log 2>&1
echo "ncu $k rc=$?"
done
