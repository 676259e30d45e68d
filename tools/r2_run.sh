cd $GRAFT_REPO_ROOT
timeout 300 python tools/dbg_tables.py > gpurun_out/r2_dbg.log 2>&1
