#!/bin/bash
# quick GPU iteration: selected parity tests + force/build timings (round 2)
cd $GRAFT_REPO_ROOT
T=${TESTS:-"tests/test_gpu_verlet.py tests/test_gpu_schedsim.py"}
timeout 900 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/rq_tests.log 2>&1; echo rc=$? >> gpurun_out/rq_tests.log
for s in ${SCHEDS:-verlet verlet_dataflow verlet_shell}; do timeout 200 python tools/time_force.py $s 50; done > gpurun_out/rq_force.log 2>&1
timeout 200 python tools/time_build.py 10 >> gpurun_out/rq_force.log 2>&1
