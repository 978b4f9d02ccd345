"""Time one decoder on EG(1023) 4 dB device-resident y (A/B helper):
python scripts/bench_alg.py ALG [weight_mode] [alpha] [lam]"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1206_3362_b200 import DecoderConfig, decode_batch, eg_ldpc
from oracle import wbf_oracle as O
alg = sys.argv[1]
wm = sys.argv[2] if len(sys.argv) > 2 else "imwbf"
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
lam = int(sys.argv[4]) if len(sys.argv) > 4 else 1
h = eg_ldpc(5)
B = 1 << 16
g = torch.Generator(device="cuda").manual_seed(1)
y = (torch.randn((B, 1023), generator=g, device="cuda") * O.ebn0_to_sigma(4.0, 781 / 1023) + 1.0).float()
cfg = DecoderConfig(alpha=alpha, k_max=100, block_len_p=31, weight_mode=wm, lam=lam)
for _ in range(2):
    decode_batch(h, y, cfg, alg)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    r = decode_batch(h, y, cfg, alg)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(json.dumps({"lib": os.path.basename(os.environ.get("FWBF_LIB", "default")), "alg": alg, "wm": wm,
                  "gbit_s": round(B * 781 / ms / 1e6, 4), "iters": float(r.iterations.float().mean())}))
