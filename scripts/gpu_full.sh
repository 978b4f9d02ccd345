#!/bin/bash
# Full measurement pass: default bench (contract line), launch list and a full
# ncu capture of the bench workload's decode kernel.  Usage: scripts/gpu_full.sh TAG
TAG=${1:-full}
mkdir -p gpurun_out
nvidia-smi -q > gpurun_out/smi_$TAG.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_full_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_full_$TAG.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
B="python bench.py --frames 65536 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/plain_full_$TAG.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_launch_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-cdecode} -s 1 -c 1 \
     -o gpurun_out/prof_full_$TAG $B > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$TAG.log
tail -n 3 gpurun_out/bench_full_$TAG.log gpurun_out/bench_ref_$TAG.log
