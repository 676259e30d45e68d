cd $GRAFT_REPO_ROOT
for s in verlet_dataflow verlet; do timeout 200 python tools/time_force.py $s 50; done > gpurun_out/r2_force.log 2>&1
CFG=cfg5 timeout 300 python tools/time_force.py verlet_dataflow 30 >> gpurun_out/r2_force.log 2>&1
CFG=cfg5 timeout 300 python tools/time_force.py verlet 30 >> gpurun_out/r2_force.log 2>&1
timeout 900 python -m pytest tests/test_gpu_verlet.py tests/test_gpu_cfg5.py tests/test_gpu_checkpoint.py -x -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
