# ncu --set full of the k_screen launches of the first (sync) c4 search
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config c4 --pairs 512 --steps 1 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:^k_screen$ -c ${1:-7} -f -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
