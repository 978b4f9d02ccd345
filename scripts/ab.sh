#!/bin/bash
# A/B timing of two builds on the same bench workload, interleaved.
# Usage: scripts/ab.sh LIB_A LIB_B [FRAMES] [ROUNDS]   (bench extra args via AB_ARGS)
A=$1; B=$2; FR=${3:-65536}; R=${4:-3}
mkdir -p gpurun_out
for r in $(seq $R); do
  for L in $A $B; do
    FWBF_LIB=$PWD/$L timeout 300 python bench.py --frames $FR --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $AB_ARGS > gpurun_out/ab.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print('$L',round(d['value'],4),round(d['ms_per_step'],3))" || tail -3 gpurun_out/ab.log
  done
done
