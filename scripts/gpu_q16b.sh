#!/bin/bash
# Q16 default: full gpu suite, then configs B/C/E A/B against the float gather
mkdir -p gpurun_out
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/q16_suite.log 2>&1
tail -6 gpurun_out/q16_suite.log
timeout 900 python scripts/bench_configs.py --only B > gpurun_out/q16_B.jsonl 2> gpurun_out/q16_cfg.err
timeout 900 python scripts/bench_configs.py --only C > gpurun_out/q16_C.jsonl 2>> gpurun_out/q16_cfg.err
FWBF_Q16=0 timeout 900 python scripts/bench_configs.py --only C > gpurun_out/f32_C.jsonl 2>> gpurun_out/q16_cfg.err
timeout 900 python scripts/bench_configs.py --only E-MLP > gpurun_out/q16_EM.jsonl 2>> gpurun_out/q16_cfg.err
FWBF_Q16=0 timeout 900 python scripts/bench_configs.py --only E-MLP > gpurun_out/f32_EM.jsonl 2>> gpurun_out/q16_cfg.err
for f in q16_B q16_C f32_C q16_EM f32_EM; do echo $f; python -c "
import json,sys
for l in open('gpurun_out/$f.jsonl'):
    d=json.loads(l); print(' ', d['config'], d.get('ebn0_db'), d.get('p'), d['frames'], round(d['info_gbit_s'],2))
"; done
