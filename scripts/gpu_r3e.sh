#!/bin/bash
# A/B (new kernel vs FWBF_NO_CDEC) at several Eb/N0, phase split, gpu suite
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r3e}
DBS=${DBS:-"4.0 4.5 5.0"} PROF=0 bash scripts/gpu_r3b.sh $TAG
for db in 4.0 5.0; do
  FWBF_PHASES=1 python bench.py --frames 262144 --steps 1 --warmup 1 --ebn0 $db --no-cpu-baseline --no-e2e 2>&1 | grep 'fwbf phases' | tail -1
done
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
  tail -n 3 gpurun_out/pytest_gpu_$TAG.log
fi
