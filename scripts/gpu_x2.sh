#!/bin/bash
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/x2_suite.log 2>&1
tail -6 gpurun_out/x2_suite.log
timeout 300 compute-sanitizer --tool memcheck --error-exitcode 3 python scripts/sanitize_small.py > gpurun_out/san_mem.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/san_mem.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 3 python scripts/sanitize_small.py > gpurun_out/san_race.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san_race.log
