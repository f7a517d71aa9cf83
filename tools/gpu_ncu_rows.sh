cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/rowbench.py 4194304 near"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_feature_distances -s 3 -c 1 -o gpurun_out/prof_rows $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/plain.log
