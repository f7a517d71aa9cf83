# Full default bench (c1 headline + c1 exhaustive, c2..c5 under "configs"), then the reference arm.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( time timeout 1700 python bench.py ) > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench_full.log
( time timeout 600 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 1500 gpurun_out/bench_ref.log
