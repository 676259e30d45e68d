cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_force.py verlet_dataflow > gpurun_out/r2_forcedf_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_force_shell -s 1 -c 1 \
  -o gpurun_out/r2_forcedf3_full python tools/prof_force.py verlet_dataflow > gpurun_out/r2_forcedf3_full.log 2>&1
