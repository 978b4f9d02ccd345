#!/bin/bash
# round-2 third session, first check: gpu suite, smoke, default bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_r2g.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r2g.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2g.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2g.log
timeout 900 python bench.py > gpurun_out/bench_r2g.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r2g.log
tail -n 2 gpurun_out/pytest_gpu_r2g.log gpurun_out/smoke_r2g.log; tail -c 3000 gpurun_out/bench_r2g.log
