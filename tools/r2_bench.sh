#!/bin/bash
# the default bench line, then the ncu launch list of the same command (cold-cache, serialised: shares only)
cd $GRAFT_REPO_ROOT
o=gpurun_out
make -s -C oracle
timeout 900 python bench.py --steps 20 --warmup 5 > $o/r2_bench.json 2> $o/r2_bench.err; echo rc=$? >> $o/r2_bench.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-schedule --no-variants --no-configs --no-link-cell > $o/r2_bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o/r2_bench_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu --no-schedule --no-variants --no-configs --no-link-cell > $o/r2_bench_ncu.log 2>&1
