#!/bin/bash
# time the force evaluation with every library variant under build/var (kernel experiments)
out=gpurun_out/var_sweep.log; : > $out
for so in build/var/*.so; do
  for sched in ${SCHEDS:-verlet}; do
    CELLSCHED_B200_LIB=$so timeout 120 python tools/time_force.py $sched ${REPS:-60} >> $out 2>&1
  done
done
