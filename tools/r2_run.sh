cd $GRAFT_REPO_ROOT
timeout 300 python tools/e2e_breakdown.py 20 > gpurun_out/r2_e2e.log 2>&1
