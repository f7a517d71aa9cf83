# usage: gpu_ncu_k.sh <kernel regex> <count> [config] -- ncu --set full of the first <count> matching launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config ${3:-c1} --steps 1 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$1" -c $2 -f -o gpurun_out/prof_k $CMD > gpurun_out/ncu_k.log 2>&1
echo "ncu rc=$?"
