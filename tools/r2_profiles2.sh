#!/bin/bash
# round-2 final captures: the dataflow kernel after the merge change; bench + its clocks
cd $GRAFT_REPO_ROOT
o=gpurun_out
timeout 300 python tools/prof_force.py verlet_dataflow > $o/r2_forcedf_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_shell -s 1 -c 1 \
  -o $o/r2_forcedf2_full python tools/prof_force.py verlet_dataflow > $o/r2_forcedf2_full.log 2>&1
timeout 300 python tools/prof_force.py verlet > $o/r2_force_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_force_shell|k_gather" \
  python tools/prof_force.py verlet > $o/r2_force_traffic.log 2>&1
