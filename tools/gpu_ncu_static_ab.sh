# ncu --set full of one search's k_screen_static launches: default library and variants/lib_$1.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config c1 --only --steps 1 --warmup 3 --no-cpu --no-allpairs"
for v in default ${1:-bound}; do
  if [ "$v" = default ]; then unset LTSG_LIB; else export LTSG_LIB=variants/lib_$v.so; fi
  $CMD > gpurun_out/plain_$v.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:k_screen_static|k_guide" -s 8 -c ${2:-8} -f -o gpurun_out/prof_static_$v $CMD > gpurun_out/ncu_$v.log 2>&1
  echo "$v ncu rc=$?"
done
