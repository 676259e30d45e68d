cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_checkpoint.py -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/racecheck_cfg1.py > gpurun_out/r2_racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2_racecheck.log
