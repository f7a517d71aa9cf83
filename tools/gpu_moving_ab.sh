# Moving-path A/B: GPU parity suite, then c4/c5 bench with the current path and with LTSG_MOVING_LEGACY=1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15
for c in ${@:-c4 c5}; do
  timeout 900 python bench.py --only --config $c --steps 5 --warmup 2 --no-cpu --no-allpairs > gpurun_out/ab_$c.log 2>&1; echo "$c new rc=$?"
  python tools/bench_table.py gpurun_out/ab_$c.log | sed -n 2p
  LTSG_MOVING_LEGACY=1 timeout 900 python bench.py --only --config $c --steps 5 --warmup 2 --no-cpu --no-allpairs > gpurun_out/ab_${c}_legacy.log 2>&1; echo "$c legacy rc=$?"
  python tools/bench_table.py gpurun_out/ab_${c}_legacy.log | sed -n 2p
done
LTSG_SYNC=1 LTSG_TRACE=1 timeout 900 python tools/trace_search.py --config c4 --pairs 2048 > gpurun_out/trace_c4_new.log 2>&1
grep "gen\|traverse\|refine" gpurun_out/trace_c4_new.log | tail -12
