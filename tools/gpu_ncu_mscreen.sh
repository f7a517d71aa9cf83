# ncu --set full (with source counters) of the two largest k_mscreen generations of a 2048-pair c4 search
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config c4 --pairs 2048 --only --steps 1 --warmup 1 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_m.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_mscreen" -s 10 -c 4 -f -o gpurun_out/prof_mscreen $CMD > gpurun_out/ncu_m.log 2>&1
echo "ncu rc=$?"
