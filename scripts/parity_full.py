"""Full-size parity of the headline workload: the bench's 2^20 frames (same
seeded generator as bench.py) decoded on the GPU and by the C oracle
(oracle/wbf_oracle.c, pinned to the reference's fixtures) on all host cores;
hard decisions, iterations, flags and flip counts compared frame by frame.
Verification script (test infrastructure), not part of the product path.

    python scripts/parity_full.py [--frames 1048576] [--ebn0 4.0] > parity.json
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.c_oracle import COracle
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from tests.golden.codebook import build_code, code_rate

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=1 << 20)
ap.add_argument("--ebn0", type=float, default=4.0)
ap.add_argument("--p", type=int, default=31)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--code", default="eg5")
ap.add_argument("--kmax", type=int, default=100)
ap.add_argument("--alg", default="fwbf")
ap.add_argument("--lam", type=int, default=1)
ap.add_argument("--weight-mode", default="imwbf")
ap.add_argument("--alpha", type=float, default=0.2)
a = ap.parse_args()

h = build_code(a.code)
n = h.n_cols
sigma = float(math.sqrt(1.0 / (2.0 * code_rate(a.code) * 10.0 ** (a.ebn0 / 10.0))))
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(a.seed * 1000003)   # bench.py, rank 0
ld = (n + 3) // 4 * 4
y = torch.empty((a.frames, ld), dtype=torch.float32, device=dev)
for s in range(0, a.frames, 1 << 16):
    y[s:min(a.frames, s + (1 << 16))].normal_(generator=g).mul_(sigma).add_(1.0)
# the bench's own layout: rows of ld floats (16-byte multiple), so the
# circulant kernels take the TMA-staged input path exactly as in bench.py
y = y[:, :n]
cfg = DecoderConfig(alpha=a.alpha, k_max=a.kmax, block_len_p=a.p, lam=a.lam, weight_mode=a.weight_mode)
t0 = time.time()
res = decode_batch(h, y, cfg, a.alg)
torch.cuda.synchronize()
tg = time.time() - t0
gz, git = res.z(), res.iterations.cpu().numpy()
gfl, gft = res.flags.cpu().numpy() & 3, res.flips_total.cpu().numpy()
yh = np.ascontiguousarray(y.cpu().numpy())
del y
t0 = time.time()
z, its, fl, ft = COracle(h).decode_batch(yh, threads=os.cpu_count(), algorithm=a.alg, alpha=a.alpha,
                                         k_max=a.kmax, p=a.p, lam=a.lam, weight_mode=a.weight_mode)
tc = time.time() - t0
bad = np.nonzero((git != its) | (gfl != fl) | (gft != ft) | np.any(gz != z, axis=1))[0]
print(json.dumps({"ld": ld, "code": a.code, "algorithm": a.alg, "lam": a.lam, "weight_mode": a.weight_mode, "alpha": a.alpha, "k_max": a.kmax, "frames": a.frames, "ebn0_db": a.ebn0, "p": a.p, "mismatched_frames": int(bad.size),
                  "first_mismatches": bad[:10].tolist(), "mean_iters": float(git.mean()),
                  "fer": float(np.mean(np.any(gz != 0, axis=1))), "gpu_s": tg, "c_oracle_s": tc,
                  "c_oracle_threads": os.cpu_count()}))
