cd $GRAFT_REPO_ROOT
make -s -C oracle
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/r2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_tests.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2_smoke.log
timeout 300 python bench.py --slab --steps 30 --warmup 5 --no-cpu > gpurun_out/r2_slab.json 2>&1; echo rc=$? >> gpurun_out/r2_slab.json
