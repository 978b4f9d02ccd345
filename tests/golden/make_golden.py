"""Generate the golden decode fixtures by running the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports `fwbf` read-only from /root/reference/pkg/src, builds each code with
this repo's constructors (checked against the reference's own EG construction
for s <= 5), draws y with the reference channel (`channel.frame_rng` +
`awgn_apply`), and records the reference decoder's outputs.  The fixtures are
the pin for both the CPU oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_parity.py); nothing reads /root/reference at test time.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import fwbf  # noqa: E402  (the reference)
from fwbf import decoders as ref_dec  # noqa: E402

from tests.golden.codebook import build_code, code_rate  # noqa: E402


def ref_matrix(code_name):
    h = build_code(code_name)
    return h, fwbf.ParityCheckMatrix(h.row_adj, h.n_cols)


def decode_ref(hr, y, alg, cfg, weight_mode):
    fn = {"fwbf": fwbf.decode_fwbf, "imwbf": fwbf.decode_imwbf, "mlp": fwbf.decode_mlp_wbf}[alg]
    if weight_mode == "mwbf":
        # F6 shim: w_nm = min1[m] for every bit of m.
        orig = ref_dec.WeightTable.edge_weights
        ref_dec.WeightTable.edge_weights = lambda self, h: self.min1[h.edge_row].copy()
        try:
            return fn(hr, y, cfg)
        finally:
            ref_dec.WeightTable.edge_weights = orig
    return fn(hr, y, cfg)


def save_case(name, code, alg, y, outs, *, alpha, k_max, lam=1, p=None,
              stall="flip-global-max", mlp_threshold=True, weight_mode="imwbf", note=""):
    B, n = y.shape
    z = np.stack([o.z_final for o in outs]).astype(np.uint8)
    log_flat, iter_len, frame_len = [], [], []
    for o in outs:
        frame_len.append(len(o.flip_log))
        for f in o.flip_log:
            iter_len.append(len(f))
            log_flat.extend(f)
    meta = dict(code=code, algorithm=alg, alpha=alpha, k_max=k_max, lam=lam, p=p,
                stall=stall, mlp_threshold=mlp_threshold, weight_mode=weight_mode,
                frames=B, n=n, dtype=str(y.dtype), note=note)
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        meta=np.array(json.dumps(meta)),
        y=y,
        z=np.packbits(z, axis=1),
        iterations=np.array([o.iterations for o in outs], np.int32),
        converged=np.array([o.converged for o in outs], np.uint8),
        stalled=np.array([o.stalled for o in outs], np.uint8),
        flips_total=np.array([o.flips_total for o in outs], np.int32),
        log_flat=np.array(log_flat, np.int32),
        log_iter_len=np.array(iter_len, np.int32),
        log_frame_len=np.array(frame_len, np.int32),
    )
    print(f"{name}: {B} frames, mean iters {np.mean([o.iterations for o in outs]):.2f}")


def channel_y(hr, ebn0, frames, seed=1, first=0, dtype=np.float32, rate=None):
    n = hr.n_cols
    sigma = fwbf.ebn0_to_sigma(ebn0, rate)
    s = fwbf.bpsk_modulate(np.zeros(n, np.uint8))
    ys = [fwbf.awgn_apply(s, sigma, fwbf.frame_rng(seed, first + i)) for i in range(frames)]
    return np.stack(ys).astype(dtype)


def case(name, code, alg, ebn0, frames, *, alpha=0.2, k_max=100, lam=1, p=None,
         stall="flip-global-max", mlp_threshold=True, weight_mode="imwbf",
         seed=1, first=0, dtype=np.float32, transform=None, y=None, note=""):
    h, hr = ref_matrix(code)
    if y is None:
        y = channel_y(hr, ebn0, frames, seed, first, dtype, code_rate(code))
    if transform is not None:
        y = transform(y)
    cfg = fwbf.DecoderConfig(alpha=alpha, k_max=k_max, lam=lam, block_len_p=p,
                             stall_policy=stall, mlp_threshold=mlp_threshold)
    outs = [decode_ref(hr, y[i], alg, cfg, weight_mode) for i in range(y.shape[0])]
    save_case(name, code, alg, y, outs, alpha=alpha, k_max=k_max, lam=lam, p=p, stall=stall,
              mlp_threshold=mlp_threshold, weight_mode=weight_mode,
              note=note or f"ebn0={ebn0} seed={seed} first={first}")


def quantize(step):
    return lambda y: (np.round(y.astype(np.float64) / step) * step).astype(y.dtype)


def main():
    # -- config B: EG(1023,781), FWBF sweep + the comparison decoders ------
    for db in (3.0, 3.5, 4.0, 4.5, 5.0):
        case(f"B_fwbf_p31_{int(db*10)}", "eg5", "fwbf", db, 12, p=31)
    case("B_fwbf_p93_40", "eg5", "fwbf", 4.0, 12, p=93)
    case("B_imwbf_40", "eg5", "imwbf", 4.0, 8)
    case("B_mlp10_40", "eg5", "mlp", 4.0, 8, lam=10)
    case("B_mlp10_all_35", "eg5", "mlp", 3.5, 6, lam=10, mlp_threshold=False)
    case("B_mwbf_40", "eg5", "imwbf", 4.0, 6, weight_mode="mwbf")
    case("B_wbf_40", "eg5", "imwbf", 4.0, 6, alpha=0.0, weight_mode="mwbf")
    case("B_fwbf_mwbf_40", "eg5", "fwbf", 4.0, 6, p=31, weight_mode="mwbf")
    case("B_fwbf_term_35", "eg5", "fwbf", 3.5, 8, p=31, stall="terminate")
    case("B_fwbf_p31_f64_40", "eg5", "fwbf", 4.0, 6, p=31, dtype=np.float64,
         note="float64 channel output, decoded without rounding")
    case("B_fwbf_p31_ties_40", "eg5", "fwbf", 4.0, 8, p=31, transform=quantize(0.125),
         note="y quantised to 1/8: many tied magnitudes and exact zeros")
    case("B_mlp_ties_40", "eg5", "mlp", 4.0, 4, lam=7, transform=quantize(0.25))
    case("B_imwbf_ties_40", "eg5", "imwbf", 4.0, 4, transform=quantize(0.25), k_max=40)
    # -- config A: (3,6) Gallager RC-free N=504 ------------------------------
    case("A_fwbf_p24_40", "gal504", "fwbf", 4.0, 32, p=24, k_max=50)
    case("A_fwbf_p24_40_a1", "gal504", "fwbf", 4.0, 16, p=24, k_max=50, alpha=1.0)
    # -- config C: EG(4095,3367) group sizes 64/128/256 -----------------------
    case("C_fwbf_p128_45", "eg6", "fwbf", 4.5, 4, p=128)
    case("C_fwbf_p64_40", "eg6", "fwbf", 4.0, 2, p=64)
    case("C_fwbf_p256_40", "eg6", "fwbf", 4.0, 2, p=256)
    # -- config D: QC(4,32) N=16384 -------------------------------------------
    case("D_fwbf_p256_50", "qc4x32", "fwbf", 5.0, 3, p=256, k_max=50)
    # -- small codes and edge cases -------------------------------------------
    case("S_eg4_fwbf_p16_30", "eg4", "fwbf", 3.0, 24, p=16, k_max=30)
    case("S_eg4_fwbf_p1_30", "eg4", "fwbf", 3.0, 12, p=1, k_max=30)
    case("S_eg4_fwbf_pN_30", "eg4", "fwbf", 3.0, 12, p=255, k_max=30)
    case("S_eg4_fwbf_pbig_30", "eg4", "fwbf", 3.0, 8, p=1000, k_max=30)
    case("S_eg4_mlp_lamN_30", "eg4", "mlp", 3.0, 6, lam=255, k_max=20)
    case("S_eg4_mlp_lam1_30", "eg4", "mlp", 3.0, 12, lam=1, k_max=30)
    case("S_eg4_fwbf_kmax1_30", "eg4", "fwbf", 3.0, 8, p=16, k_max=1)
    case("S_eg3_fwbf_p9_20", "eg3", "fwbf", 2.0, 24, p=9, k_max=10, stall="terminate")
    # noiseless, all-negative and all-zero frames
    h4, _ = ref_matrix("eg4")
    special = np.stack([np.ones(255), -np.ones(255), np.zeros(255),
                        np.where(np.arange(255) % 7 == 0, -0.5, 1.0),
                        np.where(np.arange(255) == 3, -0.0, 0.75)]).astype(np.float32)
    case("S_eg4_special", "eg4", "fwbf", 0.0, 0, p=16, k_max=10, y=special,
         note="noiseless / all negative / all zero / periodic errors / negative zero")
    # exhaustive single hard errors on EG(2,4) n=15 (SPEC acceptance 6)
    e = np.ones((15, 15), np.float32) - 1.8 * np.eye(15, dtype=np.float32)
    for alg, kw in (("fwbf", dict(p=4)), ("imwbf", {}), ("mlp", dict(lam=2))):
        case(f"S_eg2_single_{alg}", "eg2", alg, 0.0, 0, k_max=10, y=e, **kw)
    # -- reference channel: per-frame normals and _run_batch tuples ------------
    noise = {}
    for seed, frame in [(1, 0), (1, 1), (1, 127), (7, 5), (1, 1 << 40), (123456789, 3)]:
        rng = fwbf.frame_rng(seed, frame)
        noise[f"{seed}_{frame}"] = rng.standard_normal(1023)
    np.savez_compressed(os.path.join(HERE, "channel_normals.npz"), **noise)
    _, hr5 = ref_matrix("eg5")
    runs = []
    for (alg, cfg, db, start, count) in [
        ("fwbf", dict(block_len_p=31, k_max=100), 4.0, 0, 48),
        ("fwbf", dict(block_len_p=93, k_max=100), 3.5, 128, 32),
        ("mlp", dict(lam=10, k_max=100), 4.0, 0, 16),
    ]:
        sigma = fwbf.ebn0_to_sigma(db, 781 / 1023)
        res = fwbf.harness._run_batch(hr5, alg, fwbf.DecoderConfig(**cfg), sigma, 1, start, count, None)
        runs.append(dict(algorithm=alg, cfg=cfg, ebn0=db, sigma=sigma, seed=1, start=start,
                         count=count, result=list(res)))
    with open(os.path.join(HERE, "run_batch.json"), "w") as f:
        json.dump(runs, f, indent=1)
    # -- code constructions pinned against the reference ----------------------
    eg = {}
    for s in (2, 3, 4, 5):
        hr = fwbf.eg_ldpc_construct(s)
        eg[f"s{s}"] = np.asarray(hr.row_adj[0])
        eg[f"rank{s}"] = np.array(fwbf.gf2_rank(hr))
    np.savez_compressed(os.path.join(HERE, "eg_first_rows.npz"), **eg)
    print("done")


if __name__ == "__main__":
    main()
