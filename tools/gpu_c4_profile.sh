# Moving-path profile: per-generation trace of a c4 search (sync mode) and
# ncu --set full of its largest k_screen generation.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-8192}
LTSG_SYNC=1 timeout 900 python tools/trace_search.py --config c4 --pairs $P > gpurun_out/trace_c4.log 2>&1; echo "trace rc=$?"
grep "gen\|screen\|traverse\|refine\|stats" gpurun_out/trace_c4.log | tail -24
CMD="python tools/trace_search.py --config c4 --pairs ${2:-2048}"
LTSG_SYNC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_screen$ -s ${3:-5} -c 1 -f -o gpurun_out/prof_c4_big $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c4.log
