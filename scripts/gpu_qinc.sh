#!/bin/bash
# incremental QC kernel: parity tests, then config D with and without it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_explicit.py tests/test_gpu_parity.py tests/test_gpu_parity_scale.py tests/test_gpu_fuzz.py -m gpu -x -q -k "qc or QC or D or fuzz or golden" > gpurun_out/qinc_tests.log 2>&1
tail -15 gpurun_out/qinc_tests.log
timeout 600 python scripts/bench_configs.py --only D > gpurun_out/qinc_D.jsonl 2> gpurun_out/qinc_D.err
FWBF_NO_QCINC=1 timeout 600 python scripts/bench_configs.py --only D > gpurun_out/qinc_D_old.jsonl 2>> gpurun_out/qinc_D.err
cut -c1-200 gpurun_out/qinc_D.jsonl gpurun_out/qinc_D_old.jsonl
tail -3 gpurun_out/qinc_D.err
