#!/bin/bash
# Try guarded-path kernel shapes on the bench workload (65536 frames).
mkdir -p gpurun_out
for S in default 4x256 8x128 2x512; do
  if [ $S = default ]; then unset FWBF_SHAPE; else export FWBF_SHAPE=$S; fi
  timeout 300 python bench.py --frames 65536 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/shape_$S.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/shape_$S.log').read().strip().splitlines()[-1]);print('$S',round(d['value'],4),round(d['ms_per_step'],3))"
done
