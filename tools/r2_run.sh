cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=15 > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo rc=$? >> gpurun_out/r2_bench.err
