"""Filtered-metric probe: EG(1023) FWBF p=31 at 4 dB, decode time with and
without the filter (FWBF_NO_FILTER is read per launch), exact-resolution
counts, and (FWBF_PHASES=1) the per-phase cycle split on stderr."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.wbf_oracle import ebn0_to_sigma
from paper_1206_3362_b200 import DecoderConfig, decode_batch, eg_ldpc
from paper_1206_3362_b200.decoders import device_code

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
ebn0 = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
h = eg_ldpc(5)
g = torch.Generator(device="cuda").manual_seed(3)
y = (1.0 + ebn0_to_sigma(ebn0, 781 / 1023) * torch.randn((frames, 1024), generator=g, device="cuda")).float()
cfg = DecoderConfig(block_len_p=31, k_max=100)
dc = device_code(h)
MODES = {"filter": {}, "nofilter": {"FWBF_NO_FILTER": "1"}}
for mode in list(MODES) * 2:
    for k in ("FWBF_NO_FILTER", "FWBF_NO_WSEL"):
        os.environ.pop(k, None)
    os.environ.update(MODES[mode])
    dc.filter_stats(reset=True)
    r = decode_batch(h, y[:, :1023], cfg, "fwbf")
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = decode_batch(h, y[:, :1023], cfg, "fwbf")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(mode, f"{frames * 781 / dt / 1e9:.3f} Gbit/s", "iters", r.iterations.float().mean().item(),
          "stats", dc.filter_stats(reset=True), flush=True)
