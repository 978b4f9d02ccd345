#!/bin/bash
# ncu --set full of one decode launch of a bench.py workload.
# Usage: scripts/ncu_one.sh TAG <bench.py args...>
TAG=$1; shift
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $*"
$B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"decode_kernel|xdecode" -s 1 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
tail -1 gpurun_out/plain_$TAG.log | cut -c1-300
