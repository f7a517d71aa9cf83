# launch list + ncu --set full of one search's k_guide_static / k_screen_static launches (c1)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$1" ]; then export LTSG_LIB=variants/lib_$1.so; fi
CMD="python bench.py --config c1 --only --steps 2 --warmup 3 --no-cpu --no-allpairs"
$CMD > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_l.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c1.csv | head -14
ncu --set full --clock-control none --import-source on -k "regex:k_screen_static|k_guide" -s 16 -c 16 -f -o gpurun_out/prof_guide $CMD > gpurun_out/ncu_g.log 2>&1
echo "ncu rc=$?"
