cd $GRAFT_REPO_ROOT
timeout 200 python tools/time_force.py verlet 50 > gpurun_out/r2_abl.log 2>&1
for v in SLOT POS NORMW SLOTPOS; do CELLSCHED_B200_LIB=tools/experiments/abl/lib_$v.so timeout 200 python tools/time_force.py verlet 50; done >> gpurun_out/r2_abl.log 2>&1
