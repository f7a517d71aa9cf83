cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_contacts.py tests/test_gpu_broadphase.py -q -p no:cacheprovider --tb=short -rf > gpurun_out/pytest_cs.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_cs.log
