# ncu --set full of one search's k_expand_filter launches (c1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config c1 --only --steps 1 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_e.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_expand_filter" -s 16 -c 8 -f -o gpurun_out/prof_expand $CMD > gpurun_out/ncu_e.log 2>&1
echo "ncu rc=$?"
