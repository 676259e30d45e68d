#!/bin/bash
# round-2 verification: full GPU test suite, smoke, driver-style bench line
cd $GRAFT_REPO_ROOT
o=gpurun_out
make -s -C oracle
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > $o/r2_final_tests.log 2>&1; echo rc=$? >> $o/r2_final_tests.log
timeout 600 python __graft_entry__.py smoke > $o/r2_final_smoke.log 2>&1; echo rc=$? >> $o/r2_final_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $o/r2_final_bench.json 2> $o/r2_final_bench.err; echo rc=$? >> $o/r2_final_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $o/r2_final_ref.json 2>&1; echo rc=$? >> $o/r2_final_ref.json
