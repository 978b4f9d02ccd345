#!/bin/bash
# Q16 experiment: parity with the 16-bit gather on, then headline A/B
mkdir -p gpurun_out
FWBF_Q16=1 timeout 1200 python -m pytest tests/test_gpu_circ.py tests/test_gpu_filter.py tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -x -q -k "not qc and not QC" > gpurun_out/q16_tests.log 2>&1
tail -4 gpurun_out/q16_tests.log
for db in 4.0 4.5 5.0 3.0; do
for q in 0 1; do
FWBF_Q16=$q python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --ebn0 $db 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('q16=$q db=$db', round(d['value'],3), d['roofline']['filter'])"
done; done
