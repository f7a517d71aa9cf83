# Round profile, part B: ncu --set full of every k_screen_static launch of one async c1 search.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_screen_static -s 7 -c 14 -o gpurun_out/prof_static_full $CMD > gpurun_out/ncu_full_b.log 2>&1
echo "ncu rc=$?"
