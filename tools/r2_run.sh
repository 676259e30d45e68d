cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 200 python tools/time_build.py 10 > gpurun_out/r2_build.log 2>&1
timeout 200 python tools/time_force.py verlet 30 >> gpurun_out/r2_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_verlet.py tests/test_gpu_fullsize.py tests/test_gpu_cfg5.py tests/test_gpu_checkpoint.py -x -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
