#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/pytest_r2u.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2u.log
timeout 1200 python scripts/bench_configs.py > gpurun_out/configs_r2u.jsonl 2> gpurun_out/configs_r2u.err
timeout 600 python bench.py > gpurun_out/bench_r2u.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r2u.log 2>&1
