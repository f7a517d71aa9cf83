cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$1" -c $2 -o gpurun_out/prof_k $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
