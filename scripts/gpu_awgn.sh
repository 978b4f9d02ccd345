#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_noise.py tests/test_gpu_api_r2.py tests/test_gpu_dist.py tests/test_gpu_parity_scale.py -m gpu -x -q -k "noise or awgn or run_point or E or shard or chunk or dist or experiment or sweep" 2>&1 | tail -3
python scripts/bench_configs.py --only E 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['frames'], round(d['info_gbit_s'],2))"
