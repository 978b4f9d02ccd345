"""One MLP-WBF (lambda = 10) decode of 65,536 EG(1023) frames at 4 dB (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1206_3362_b200 import DecoderConfig, decode_batch
from tests.golden.codebook import build_code, code_rate

h = build_code("eg5")
sig = (1.0 / (2.0 * code_rate("eg5") * 10 ** 0.4)) ** 0.5
g = torch.Generator(device="cuda").manual_seed(1)
y = torch.randn((65536, 1024), device="cuda", generator=g).mul_(sig).add_(1.0)[:, :1023]
for _ in range(2):
    r = decode_batch(h, y, DecoderConfig(lam=10, k_max=100), "mlp")
torch.cuda.synchronize()
print("ok", r.iterations.float().mean().item())
