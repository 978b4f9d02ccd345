#!/bin/bash
# new filtered circulant kernel: quick A/B against decode_kernel MODE 2, then the gpu suite
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for db in 4.0 5.0; do
  for rep in 1 2; do
    for envs in "FWBF_NO_CDEC=1" "FWBF_DUMMY=1"; do
      env $envs timeout 300 python bench.py --steps 3 --warmup 3 --ebn0 $db --no-cpu-baseline --no-e2e > gpurun_out/ab_r3a.log 2>&1
      python -c "import json,sys; d=json.loads(open('gpurun_out/ab_r3a.log').read().strip().splitlines()[-1]); print('$envs', $db, round(d['value'],3), round(d['ms_per_step'],2), d['config']['mean_iters'], d['config']['fer'])" || tail -5 gpurun_out/ab_r3a.log
    done
  done
done
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_r3a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r3a.log
tail -n 30 gpurun_out/pytest_gpu_r3a.log
