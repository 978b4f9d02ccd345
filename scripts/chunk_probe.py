"""Where the e2e leg's 7 % goes: the headline batch decoded device-resident in one launch,
in 8 chunks of 2^17 frames, and in the pipeline's ramp (2^13 ... 2^17), no copies."""
import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1206_3362_b200 import DecoderConfig, decode_batch, eg_ldpc
from oracle import wbf_oracle as O
h = eg_ldpc(5); B = 1 << 20
g = torch.Generator(device="cuda").manual_seed(1)
y = torch.zeros((B, 1024), dtype=torch.float32, device="cuda")
y[:, :1023] = 1.0 + O.ebn0_to_sigma(4.0, 781 / 1023) * torch.randn((B, 1023), generator=g, device="cuda")
yv = y[:, :1023]
cfg = DecoderConfig(block_len_p=31, k_max=100)
def run(chunks):
    torch.cuda.synchronize(); t = time.perf_counter()
    f0 = 0
    for c in chunks:
        decode_batch(h, yv[f0:f0 + c], cfg, "fwbf"); f0 += c
    torch.cuda.synchronize(); return (time.perf_counter() - t) * 1e3
ramp = [8192, 16384, 32768, 65536] + [131072] * 7 + [8192 * 1]
ramp[-1] = B - sum(ramp[:-1])
for name, ch in (("one launch", [B]), ("8 x 2^17", [131072] * 8), ("pipeline ramp", ramp), ("64 x 2^14", [16384] * 64)):
    run(ch); ts = [run(ch) for _ in range(3)]
    print(name, [round(t, 2) for t in ts], "ms; Gbit/s", round(B * 781 / min(ts) / 1e6, 3))
