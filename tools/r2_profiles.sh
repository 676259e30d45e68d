#!/bin/bash
# Round-2 profiles (run under gpurun): edge-case tests, the eager Verlet step's launch list,
# full ncu captures of the Verlet force kernel (buffered + dataflow) and the list builder.
cd $GRAFT_REPO_ROOT
o=gpurun_out
make -s -C oracle
timeout 600 python -m pytest tests/test_gpu_edges.py -q -p no:cacheprovider > $o/r2_edges.log 2>&1; echo rc=$? >> $o/r2_edges.log
timeout 300 python tools/prof_step.py 20 > $o/r2_step_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $o/r2_step_launches.csv python tools/prof_step.py 20 > $o/r2_step_ncu.log 2>&1
timeout 300 python tools/prof_force.py verlet > $o/r2_force_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_shell -s 1 -c 1 \
  -o $o/r2_force_full python tools/prof_force.py verlet > $o/r2_force_full.log 2>&1
timeout 300 python tools/prof_force.py verlet_dataflow > $o/r2_forcedf_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_shell -s 1 -c 1 \
  -o $o/r2_forcedf_full python tools/prof_force.py verlet_dataflow > $o/r2_forcedf_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verlet_build -c 1 \
  -o $o/r2_build_full python tools/prof_force.py verlet > $o/r2_build_full.log 2>&1
