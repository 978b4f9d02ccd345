#!/bin/bash
# ncu --set full of the headline decode kernel with source; exports the SASS and
# CUDA source pages as CSV.  Usage: scripts/gpu_prof.sh TAG [bench args]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=$1; shift
mkdir -p gpurun_out
B="python bench.py --frames 16384 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $*"
$B > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"${KRE:-decode_kernel|xdecode|qdecode}" -s 1 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$TAG.csv 2>/dev/null
tail -1 gpurun_out/plain_$TAG.log | cut -c1-400; tail -2 gpurun_out/ncu_$TAG.log
