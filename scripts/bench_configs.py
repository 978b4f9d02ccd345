"""Throughput of every BASELINE.json configuration (A-E) on one B200.

Writes one JSON line per (config, decoder, Eb/N0) to stdout; the contract
line for the headline workload stays in bench.py.  Inputs are seeded
synthetic AWGN frames of each config's shape (device-resident float32 y for
A-D; on-device reference-channel noise for E).  Timing: CUDA events on the
launching stream around `steps` decode calls after `warmup` calls.

    python scripts/bench_configs.py [--quick] > profiles/rN_configs.jsonl
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_1206_3362_b200 import DecoderConfig, _native as nat  # noqa: E402
from paper_1206_3362_b200.decoders import BatchResult, _outputs, device_code, make_params  # noqa: E402
from tests.golden.codebook import build_code, code_k, code_rate  # noqa: E402


def sigma_of(code, ebn0):
    return math.sqrt(1.0 / (2.0 * code_rate(code) * 10.0 ** (ebn0 / 10.0)))


def run_y(code, alg, cfg, ebn0, frames, steps, warmup, seed=1):
    h = build_code(code)
    n = h.n_cols
    ld = (n + 3) // 4 * 4
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(seed)
    y = torch.empty((frames, ld), dtype=torch.float32, device=dev)
    for s in range(0, frames, 1 << 16):
        y[s:s + (1 << 16)].normal_(generator=g).mul_(sigma_of(code, ebn0)).add_(1.0)
    dc = device_code(h, 0)
    prm = make_params(cfg, alg)
    zw = (n + 31) // 32
    res = BatchResult(n=n, z_bits=torch.zeros((frames, zw), dtype=torch.int32, device=dev),
                      iterations=torch.zeros(frames, dtype=torch.int32, device=dev),
                      flags=torch.zeros(frames, dtype=torch.uint8, device=dev),
                      flips_total=torch.zeros(frames, dtype=torch.int32, device=dev),
                      bit_errors=torch.zeros(frames, dtype=torch.int32, device=dev),
                      counters=torch.zeros(nat.NCOUNTERS, dtype=torch.int64, device=dev))
    res.iter_hist = torch.zeros(cfg.k_max + 1, dtype=torch.int64, device=dev)
    out = _outputs(res)
    st = torch.cuda.current_stream(dev)
    L = nat.lib()

    def step():
        res.counters.zero_()
        res.iter_hist.zero_()
        nat.check(L.fwbf_decode_f32(dc.handle, C.byref(prm), C.c_void_p(y.data_ptr()), frames, ld,
                                    C.byref(out), C.c_void_p(st.cuda_stream)), "decode")
    return _time(step, steps, warmup, res, frames, code, h)


def run_awgn(code, alg, cfg, ebn0, frames, steps, warmup, noise="f32", seed=1):
    from paper_1206_3362_b200.decoders import decode_awgn
    h = build_code(code)
    sigma = sigma_of(code, ebn0)
    holder = {}

    def step():
        holder["r"] = decode_awgn(h, cfg, alg, seed, 0, frames, sigma, noise=noise)
    step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    return _summ(holder["r"], frames, ms, code, h, device_noise=True)


def _time(step, steps, warmup, res, frames, code, h):
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    return _summ(res, frames, ev0.elapsed_time(ev1) / steps, code, h)


def _peaks():
    props = torch.cuda.get_device_properties(0)
    try:
        mp = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except OSError:
        mp = {}
    return props.multi_processor_count, mp.get("sm_max_mhz", 1965.0), mp.get("hbm_gbs", 6548.2)


def _summ(res, frames, ms, code, h, device_noise=False):
    c = res.counters.cpu().numpy()
    fr = int(c[nat.CNT_FRAMES])
    it = c[nat.CNT_ITER_SUM] / fr
    sms, mhz, hbm = _peaks()
    ev = h.n_edges * (1 + it) * frames / (ms / 1e3)
    zw = (h.n_cols + 31) // 32
    bpf = (0 if device_noise else 4 * h.n_cols) + 4 * zw + 8   # SURVEY 8(d) algorithmic bytes per frame
    out = {"frames": frames, "ms_per_step": ms, "info_gbit_s": frames * code_k(code) / (ms / 1e3) / 1e9,
           "frames_per_s": frames / (ms / 1e3), "mean_iters": float(it),
           "fer": float(c[nat.CNT_WORD_ERRORS] / fr), "ber": float(c[nat.CNT_BIT_ERRORS] / (fr * h.n_cols)),
           "ordered_frames": int(c[nat.CNT_ORDERED_FRAMES]),
           "edge_visits_per_s": ev,
           # the binding roofline of SURVEY 8(d): one fp64 add per lane per clock
           "roofline": {"bound": "issue", "achieved": ev, "peak": sms * 64 * mhz * 1e6, "unit": "edge-visits/s",
                        "frac": ev / (sms * 64 * mhz * 1e6),
                        "hbm": {"bytes_per_frame": bpf, "achieved_GBps": bpf * frames / (ms / 1e3) / 1e9,
                                "frac": bpf * frames / (ms / 1e3) / 1e9 / hbm}}}
    if getattr(res, "iter_hist", None) is not None:
        out["iter_hist"] = [int(v) for v in res.iter_hist.cpu().tolist()]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    q = a.quick
    jobs = []
    # A: (3,6) Gallager N=504, 4 dB, FWBF K_max 50, 10,000 frames
    jobs.append(("A", "gal504", "fwbf", DecoderConfig(block_len_p=24, k_max=50), 4.0, 10000, "y"))
    # B: EG(1023,781) sweep 3.0-5.0 dB, FWBF p=31/93 and the comparison decoders at 4 dB
    fb = 1 << (16 if q else 20)
    for db in (3.0, 3.5, 4.0, 4.5, 5.0):
        jobs.append(("B", "eg5", "fwbf", DecoderConfig(block_len_p=31, k_max=100), db, fb, "y"))
    jobs.append(("B", "eg5", "fwbf", DecoderConfig(block_len_p=93, k_max=100), 4.0, fb, "y"))
    jobs.append(("B-IMWBF", "eg5", "imwbf", DecoderConfig(k_max=100), 4.0, fb >> 2, "y"))
    jobs.append(("B-MWBF", "eg5", "imwbf", DecoderConfig(k_max=100, weight_mode="mwbf"), 4.0, fb >> 2, "y"))
    jobs.append(("B-WBF", "eg5", "imwbf", DecoderConfig(k_max=100, alpha=0.0, weight_mode="mwbf"), 4.0,
                 fb >> 2, "y"))
    # C: EG(4095,3367), 3.5-4.5 dB, group sizes 64/128/256, 2^18 frames
    fc = 1 << (14 if q else 18)
    for pp in (64, 128, 256):
        for db in (3.5, 4.0, 4.5):
            jobs.append(("C", "eg6", "fwbf", DecoderConfig(block_len_p=pp, k_max=100), db, fc, "y"))
    # D: QC(4,32) N=16384, 5 dB, K_max 50, 2^16 frames
    jobs.append(("D", "qc4x32", "fwbf", DecoderConfig(block_len_p=256, k_max=50), 5.0,
                 1 << (12 if q else 16), "y"))
    # E: EG(1023) 4 dB, on-device reference-channel noise, batch 2^10..2^24, FWBF vs MLP
    for lg in (10, 14, 18, 20) if q else (10, 12, 14, 16, 18, 20, 22, 24):
        jobs.append(("E", "eg5", "fwbf", DecoderConfig(block_len_p=31, k_max=100), 4.0, 1 << lg, "awgn"))
        if lg <= 20:
            jobs.append(("E-MLP", "eg5", "mlp", DecoderConfig(lam=10, k_max=100), 4.0, 1 << lg, "awgn"))
    for name, code, alg, cfg, db, frames, src in jobs:
        if a.only and not name.startswith(a.only):
            continue
        steps, warm = (3, 2) if frames >= (1 << 16) else (10, 3)
        r = (run_y if src == "y" else run_awgn)(code, alg, cfg, db, frames, steps, warm)
        r.update(config=name, code=code, algorithm=alg, ebn0_db=db, p=cfg.block_len_p, lam=cfg.lam,
                 k_max=cfg.k_max, alpha=cfg.alpha, weight_mode=cfg.weight_mode,
                 input="device float32 y" if src == "y" else "on-device numpy-stream noise (f32)")
        print(json.dumps(r), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
