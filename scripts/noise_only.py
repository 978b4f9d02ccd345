"""Time decode_awgn (reference-channel noise kernel + decode) on EG(1023) 4 dB;
run under different FWBF_NOISE_GRID / FWBF_NOISE_T to tune the noise kernel."""
import math, sys, time
sys.path.insert(0, '.')
import torch
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate
h = build_code('eg5'); sigma = math.sqrt(1 / (2 * code_rate('eg5') * 10 ** 0.4))
cfg = DecoderConfig(block_len_p=31, k_max=100)
F = 1 << 18
for noise in ('f32', 'f64'):
    decode_awgn(h, cfg, 'fwbf', 1, 0, F, sigma, noise=noise); torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        t = time.perf_counter(); decode_awgn(h, cfg, 'fwbf', 1, 0, F, sigma, noise=noise); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(noise, 'ms', round(min(ts) * 1e3, 2), 'Gbit/s', round(F * 781 / min(ts) / 1e9, 3), flush=True)
