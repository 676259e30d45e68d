#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_sched.py -x -q -p no:cacheprovider > gpurun_out/qs_tests.log 2>&1; echo rc=$? >> gpurun_out/qs_tests.log
timeout 300 python -c "
import sys, json, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.schedule_report(torch, cpu=False)))" > gpurun_out/qs_sched.log 2>&1
