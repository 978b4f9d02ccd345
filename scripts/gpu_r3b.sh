#!/bin/bash
# A/B of the filtered circulant kernel vs decode_kernel MODE 2 + ncu capture
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r3b}
for db in ${DBS:-4.0 5.0}; do
  for rep in 1 2; do
    for envs in "FWBF_NO_CDEC=1" "FWBF_DUMMY=1"; do
      env $envs timeout 300 python bench.py --steps 3 --warmup 3 --ebn0 $db --no-cpu-baseline --no-e2e $BARGS > gpurun_out/ab_$TAG.log 2>&1
      python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$TAG.log').read().strip().splitlines()[-1]); print('$envs', $db, round(d['value'],3), round(d['ms_per_step'],2), d['config']['mean_iters'], d['config']['fer'])" || tail -5 gpurun_out/ab_$TAG.log
    done
  done
done
if [ "${TESTS:-0}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  tail -n 3 gpurun_out/pytest_gpu_$TAG.log
fi
if [ "${PROF:-1}" = "1" ]; then KRE=cdecode bash scripts/gpu_prof.sh $TAG > /dev/null 2>&1; tail -1 gpurun_out/ncu_$TAG.log; fi
