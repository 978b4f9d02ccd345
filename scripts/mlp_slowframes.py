"""Locate frames that are slow on the filtered MLP path (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200.decoders import device_code
from tests.golden.codebook import build_code, code_rate

h = build_code("eg5")
sig = (1.0 / (2.0 * code_rate("eg5") * 10 ** 0.4)) ** 0.5
cfg = DecoderConfig(lam=10, k_max=100)
dc = device_code(h)
g = torch.Generator(device="cuda").manual_seed(1)
y = torch.randn((65536, 1024), device="cuda", generator=g).mul_(sig).add_(1.0)[:, :1023]


def t(sl, reps=2):
    best = 1e9
    for _ in range(reps):
        dc.filter_stats(reset=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = decode_batch(h, y[sl], cfg, "mlp")
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, r, dc.filter_stats(reset=True)


for c in range(16):
    dt, r, st = t(slice(4096 * c, 4096 * (c + 1)))
    print(f"chunk {c:2d}: {dt * 1e3:7.2f} ms exact {st}", flush=True)
worst = max(range(16), key=lambda c: t(slice(4096 * c, 4096 * (c + 1)))[0])
lo = 4096 * worst
for s in range(0, 4096, 256):
    dt, r, st = t(slice(lo + s, lo + s + 256))
    if dt > 0.004:
        for f in range(lo + s, lo + s + 256):
            d1, r1, s1 = t(slice(f, f + 1), 1)
            if d1 > 0.002:
                print(f"slow frame {f}: {d1 * 1e3:.2f} ms iters {int(r1.iterations[0])} exact {s1} "
                      f"min|y| {y[f].abs().min().item():.3e} max|y| {y[f].abs().max().item():.3f}", flush=True)
