"""Small decodes of every new kernel path for compute-sanitizer (memcheck / racecheck):
    compute-sanitizer --tool racecheck python scripts/sanitize_small.py
Each result is also checked against the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import wbf_oracle as O
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from tests.golden.codebook import build_code, code_rate

rng = np.random.default_rng(3)
for code, p, kmax, db, frames, alg in (("eg5", 31, 30, 4.0, 40, "fwbf"), ("eg5", 93, 20, 4.0, 16, "fwbf"),
                                       ("eg4", 17, 20, 4.0, 16, "fwbf"), ("eg5", 31, 20, 4.0, 16, "mlp"),
                                       ("qc4x32", 256, 12, 5.0, 6, "fwbf"), ("qc4x32", 64, 12, 5.5, 6, "fwbf"),
                                       ("gal504", 24, 30, 4.0, 40, "fwbf")):
    h = build_code(code)
    y = (1.0 + O.ebn0_to_sigma(db, code_rate(code)) * rng.standard_normal((frames, h.n_cols))).astype(np.float32)
    y[1] = np.round(y[1] * 2) / 2
    cfg = DecoderConfig(block_len_p=p, k_max=kmax, lam=5) if alg == "fwbf" else DecoderConfig(lam=5, k_max=kmax)
    r = decode_batch(h, y, cfg, alg, flip_log=True, device="cuda:0")
    torch.cuda.synchronize()
    g = O.Graph.of(h)
    its = r.iterations.cpu().numpy()
    z = r.z()
    for i in range(min(frames, 6)):
        ref = O.decode(g, y[i], alg, alpha=cfg.alpha, k_max=kmax, p=p, lam=5)
        assert its[i] == ref.iterations and np.array_equal(z[i], ref.z), (code, p, alg, i)
    print(code, p, alg, nat.last_kernel(), "ok", its[:6])
