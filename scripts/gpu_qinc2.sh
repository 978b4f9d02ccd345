#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_explicit.py -m gpu -x -q -k "qc" > gpurun_out/qinc_tests.log 2>&1
tail -3 gpurun_out/qinc_tests.log
for i in 1 2; do
timeout 600 python scripts/bench_configs.py --only D 2>> gpurun_out/qinc_D.err | cut -c1-120
FWBF_NO_QCPREFETCH=1 timeout 600 python scripts/bench_configs.py --only D 2>> gpurun_out/qinc_D.err | cut -c1-120
done
