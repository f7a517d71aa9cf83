# ncu --set full of the static screen + SAT filter launches of one async c1 search
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_g.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_screen_static|k_sat_filter" -s ${1:-14} -c ${2:-12} -o gpurun_out/prof_gen $CMD > gpurun_out/ncu_gen.log 2>&1
echo "ncu rc=$?"
