cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_schedsim.py -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
