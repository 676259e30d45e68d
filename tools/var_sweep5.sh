#!/bin/bash
# force + build timing of every variant under build/var on cfg2 and cfg5 (kernel experiments)
out=gpurun_out/var_sweep.log; : > $out
for so in build/var/*.so; do
  CELLSCHED_B200_LIB=$so timeout 120 python tools/time_force.py verlet ${REPS:-60} >> $out 2>&1
  CELLSCHED_B200_LIB=$so CFG=cfg5 timeout 300 python tools/time_force.py verlet ${REPS5:-20} >> $out 2>&1
done
