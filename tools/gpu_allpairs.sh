# allpairs kernel: parity tests, microbench of variant libraries, ncu of the default tile kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_allpairs.py -q -x -p no:cacheprovider --tb=short > gpurun_out/pytest_allpairs.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_allpairs.log
timeout 300 python tools/allpairs_bench.py 16 tile,staged 2>&1 | tail -2
for v in variants/lib_*.so; do LTSG_LIB=$v timeout 300 python tools/allpairs_bench.py 16 tile 2>&1 | tail -1 | sed "s|^|$v |"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_allpairs_tile -c 1 -f -o gpurun_out/prof_allpairs python tools/allpairs_bench.py 4 tile > gpurun_out/ncu_allpairs.log 2>&1; echo "ncu rc=$?"
