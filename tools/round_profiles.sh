#!/bin/bash
# Round profiles: default bench, the bench's launch list under ncu, full captures of the
# Verlet force kernel and the list builder (run under gpurun; outputs in gpurun_out/)
o=gpurun_out
timeout 900 python bench.py > $o/bench_full.log 2>&1; echo rc=$? >> $o/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file $o/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu --no-schedule > $o/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_force_shell -s 1 -c 1 \
  -o $o/force_full python tools/prof_force.py verlet > $o/force_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_verlet_build -c 1 \
  -o $o/build_full python tools/prof_force.py verlet > $o/build_full.log 2>&1
