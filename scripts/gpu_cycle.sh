#!/bin/bash
# One build->measure cycle on the GPU box: GPU tests, a short bench, an ncu
# capture of the decode kernel.  Usage: scripts/gpu_cycle.sh TAG [FRAMES]
TAG=${1:-x}; FR=${2:-65536}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --frames $FR --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
B="python bench.py --frames 16384 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
if [ "${NCU:-1}" = "1" ]; then
  $B > gpurun_out/plain_$TAG.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
     -k regex:decode_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
fi
tail -n 2 gpurun_out/pytest_gpu_$TAG.log
python - "$TAG" <<'PY'
import json,sys
try:
    d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
    print("value",d["value"],"ms",d["ms_per_step"],"iters",d["config"]["mean_iters"],"e2e",d["e2e"]["value"] if d.get("e2e") else None)
except Exception as e: print("bench parse failed",e)
PY
