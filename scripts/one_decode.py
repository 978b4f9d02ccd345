import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_1206_3362_b200 import DecoderConfig, decode_batch, eg_ldpc
h=eg_ldpc(5); rng=np.random.default_rng(1)
y=(1+0.55*rng.standard_normal((65536,1023))).astype(np.float32)
try:
    r=decode_batch(h,y,DecoderConfig(block_len_p=31,k_max=20),"fwbf"); torch.cuda.synchronize(); print("ok", r.iterations.float().mean().item())
except Exception as e: print("ERR", str(e)[:300])
