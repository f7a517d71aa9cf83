# c4 bench (full 8192 pairs) on the current moving path, then ncu --set full of
# the largest k_mscreen generation (2048 pairs, sync mode) and the per-gen trace.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --only --config c4 --steps 5 --warmup 2 --no-cpu --no-allpairs > gpurun_out/c4_new.log 2>&1; echo "c4 rc=$?"
python tools/bench_table.py gpurun_out/c4_new.log | sed -n 2p
tail -3 gpurun_out/c4_new.log | grep -i error
LTSG_SYNC=1 LTSG_TRACE=1 timeout 900 python tools/trace_search.py --config c4 --pairs 2048 > gpurun_out/trace_c4_new.log 2>&1
grep "gen\|traverse\|refine\|stats" gpurun_out/trace_c4_new.log | tail -12
CMD="python tools/trace_search.py --config c4 --pairs 2048"
LTSG_SYNC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_mscreen$ -s 5 -c 1 -f -o gpurun_out/prof_mscreen $CMD > gpurun_out/ncu_ms.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_ms.log
LTSG_SYNC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_mexact$ -s 5 -c 1 -f -o gpurun_out/prof_mexact $CMD > gpurun_out/ncu_mx.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_mx.log
