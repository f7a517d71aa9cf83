cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config c4 --pairs 256 --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_screen" -s 5 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
