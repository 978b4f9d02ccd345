#!/bin/bash
# Per-phase cycle split (FWBF_PHASES=1) for configs A, C, D (quick sizes).
mkdir -p gpurun_out
export FWBF_PHASES=1
for C in A C D; do
  timeout 600 python scripts/bench_configs.py --quick --only $C > gpurun_out/ph_$C.jsonl 2> gpurun_out/ph_$C.err
  echo "== $C"; cat gpurun_out/ph_$C.jsonl | cut -c1-200; sort gpurun_out/ph_$C.err | uniq -c | sort -rn | head -12
done
