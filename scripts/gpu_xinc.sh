#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_explicit.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -k "warp or gal or A or fuzz or golden or dv4" > gpurun_out/xinc_tests.log 2>&1
tail -6 gpurun_out/xinc_tests.log
for i in 1 2; do
python scripts/bench_configs.py --only A 2>/dev/null | cut -c1-110
FWBF_NO_XINC=1 python scripts/bench_configs.py --only A 2>/dev/null | cut -c1-110
done
python - <<'PY'
import sys, time; sys.path.insert(0,'.')
import numpy as np, torch, os
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from tests.golden.codebook import build_code, code_rate
from oracle import wbf_oracle as O
h=build_code("gal504"); rng=np.random.default_rng(1)
y=torch.from_numpy((1+O.ebn0_to_sigma(4.0,code_rate("gal504"))*rng.standard_normal((1<<20,504))).astype(np.float32)).cuda()
cfg=DecoderConfig(block_len_p=24,k_max=50)
for env in (None,"1",None,"1"):
    if env: os.environ["FWBF_NO_XINC"]=env
    else: os.environ.pop("FWBF_NO_XINC",None)
    decode_batch(h,y,cfg,"fwbf"); torch.cuda.synchronize(); t=time.time()
    for _ in range(3): r=decode_batch(h,y,cfg,"fwbf")
    torch.cuda.synchronize(); dt=(time.time()-t)/3
    print(nat.last_kernel(), "2^20 frames", round((1<<20)*252/dt/1e9,3), "Gbit/s", float(r.iterations.float().mean()))
PY
