"""A/B helper: time the float64 (ordered, exact-replay) path on EG(1023) FWBF p=31."""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1206_3362_b200 import DecoderConfig, decode_batch, eg_ldpc
h = eg_ldpc(5)
g = torch.Generator(device="cuda").manual_seed(1)
B = 16384
y = (torch.randn((B, 1023), generator=g, device="cuda", dtype=torch.float64) * 0.5106 + 1.0)
cfg = DecoderConfig(alpha=0.2, k_max=100, block_len_p=31)
for _ in range(2):
    decode_batch(h, y, cfg, "fwbf")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    r = decode_batch(h, y, cfg, "fwbf")
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(json.dumps({"lib": os.environ.get("FWBF_LIB"), "f64_gbit_s": B * 781 / ms / 1e6, "ms": ms}))
