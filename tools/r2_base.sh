cd $GRAFT_REPO_ROOT
for s in verlet verlet_shell verlet_dataflow buffered dataflow shell loopex; do timeout 200 python tools/time_force.py $s 50; done > gpurun_out/r2_base_force.log 2>&1
timeout 200 python tools/time_build.py 20 > gpurun_out/r2_base_build.log 2>&1
timeout 200 python tools/time_step.py > gpurun_out/r2_base_step.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/r2_base_step.log
