#!/bin/bash
# quick GPU check of the Verlet path: parity tests, short bench, force-kernel time
set -x
timeout 600 python -m pytest tests/test_gpu_verlet.py tests/test_gpu_lj.py tests/test_gpu_slab.py -x -q -p no:cacheprovider > gpurun_out/qv_tests.log 2>&1; echo rc=$? >> gpurun_out/qv_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu --no-link-cell > gpurun_out/qv_bench.log 2>&1; echo rc=$? >> gpurun_out/qv_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_force_shell|k_verlet_build|k_vl_recode|k_gather" -c 12 python tools/prof_force.py verlet > gpurun_out/qv_ncu.log 2>&1
