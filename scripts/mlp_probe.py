"""MLP-WBF on the filtered circulant kernel vs decode_kernel MODE 0: time,
exact-decision counts and phase split for a few batch sizes (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.decoders import device_code
from tests.golden.codebook import build_code, code_rate

h = build_code("eg5")
sig = (1.0 / (2.0 * code_rate("eg5") * 10 ** 0.4)) ** 0.5
cfg = DecoderConfig(lam=int(os.environ.get("LAM", "10")), k_max=100)
dc = device_code(h)
for frames in [int(x) for x in os.environ.get("FRAMES", "16384 65536 262144").split()]:
    g = torch.Generator(device="cuda").manual_seed(1)
    y = torch.randn((frames, 1024), device="cuda", generator=g).mul_(sig).add_(1.0)[:, :1023]
    for env in ("", "FWBF_NO_CDEC"):
        if env:
            os.environ[env] = "1"
        for rep in range(3):
            dc.filter_stats(reset=True)
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = decode_batch(h, y, cfg, "mlp")
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        st = dc.filter_stats(reset=True)
        print(f"frames {frames} {'mode0' if env else 'cdec '} {dt * 1e3:8.2f} ms  iters {r.iterations.float().mean().item():.2f}  "
              f"exact {st}  kern {nat.last_kernel()}", flush=True)
        if env:
            del os.environ[env]
