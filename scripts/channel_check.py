"""Count device-vs-numpy channel mismatches over many frames (reference stream replay).

    python scripts/channel_check.py FRAMES [SEED]
"""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import wbf_oracle as O  # noqa: E402  (checker only)
from paper_1206_3362_b200 import DecoderConfig  # noqa: E402
from paper_1206_3362_b200.decoders import decode_awgn  # noqa: E402
from tests.golden.codebook import build_code, code_rate  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h = build_code("eg5")
sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
bad_vals = bad_frames = 0
chunk = 4096
for s in range(0, frames, chunk):
    n = min(chunk, frames - s)
    res = decode_awgn(h, DecoderConfig(block_len_p=31, k_max=1), "fwbf", seed, s, n, sigma, return_y=True)
    y = res.y.cpu().numpy()
    ref = np.stack([O.channel_frame(np.zeros(1023, np.uint8), sigma, seed, s + i) for i in range(n)])
    d = y != ref
    bad_vals += int(d.sum())
    bad_frames += int(d.any(axis=1).sum())
print(f"frames {frames} values {frames * 1023} mismatched values {bad_vals} mismatched frames {bad_frames}")
