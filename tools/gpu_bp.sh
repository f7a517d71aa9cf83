cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_broadphase.py -q -p no:cacheprovider --tb=short -rf > gpurun_out/pytest_bp.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_bp.log
timeout 600 python tools/bp_quick.py 2>&1 | grep -v Warn | tail -5
