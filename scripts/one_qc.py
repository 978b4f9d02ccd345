"""One decode of config D (QC(16384) FWBF p=256, 5 dB) for ncu.  Usage: one_qc.py [frames]"""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from tests.golden.codebook import build_code, code_rate
from oracle import wbf_oracle as O
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
h = build_code("qc4x32")
rng = np.random.default_rng(1)
y = torch.from_numpy((1 + O.ebn0_to_sigma(5.0, code_rate("qc4x32")) * rng.standard_normal((frames, h.n_cols))).astype(np.float32)).cuda()
for _ in range(2):
    r = decode_batch(h, y, DecoderConfig(block_len_p=256, k_max=50), "fwbf", device="cuda:0")
    torch.cuda.synchronize()
print("ok", r.iterations.float().mean().item(), r.flips_total.float().mean().item())
