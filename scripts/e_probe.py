import sys, time, math; sys.path.insert(0, '.')
import torch
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate
h = build_code('eg5'); sigma = math.sqrt(1 / (2 * code_rate('eg5') * 10 ** 0.4))
for alg, cfg, lgs in (("fwbf", DecoderConfig(block_len_p=31, k_max=100), (18, 20, 22)), ("mlp", DecoderConfig(lam=10, k_max=100), (18, 20))):
    for lg in lgs:
        F = 1 << lg
        decode_awgn(h, cfg, alg, 1, 0, F, sigma, noise="f32"); torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            t = time.perf_counter(); decode_awgn(h, cfg, alg, 1, 0, F, sigma, noise="f32"); torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        print(alg, lg, round(F * 781 / min(ts) / 1e9, 3), flush=True)
