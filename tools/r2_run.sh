cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 1500 python -m pytest tests/test_gpu_schedsim.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -s --durations=20 > gpurun_out/rq_tests.log 2>&1; echo rc=$? >> gpurun_out/rq_tests.log
