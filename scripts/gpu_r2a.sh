#!/bin/bash
# round-2 GPU check: full -m gpu suite (timings), bench, reference arm
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=40 -p no:cacheprovider > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2a.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_r2a.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_r2a.log 2>&1
echo "ref rc=$?" >> gpurun_out/bench_ref_r2a.log
