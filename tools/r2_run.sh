cd $GRAFT_REPO_ROOT
timeout 600 python tools/time_build.py 10 > gpurun_out/r2_build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_vb_" -c 2 python tools/time_build.py 1 > gpurun_out/r2_ncu_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_verlet.py -x -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
