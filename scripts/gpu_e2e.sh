#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_host_pipeline.py tests/test_c_client.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
python bench.py --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))"
done
for ch in 65536 262144; do python bench.py --no-cpu-baseline --steps 3 --warmup 3 --e2e-chunk $ch 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print(d['e2e']['chunk_frames'], round(d['value'],3), round(d['e2e']['value'],3))"; done
