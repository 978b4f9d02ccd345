"""Parity at scale: every BASELINE config, tens of thousands of frames, CUDA vs
the C oracle (oracle/wbf_oracle.c, itself pinned to the reference fixtures).
Bit-exact per frame: hard decisions, iterations, converged/stalled, flip count."""

import numpy as np
import pytest

from oracle import wbf_oracle as O
from oracle.c_oracle import COracle
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate

pytestmark = pytest.mark.gpu

CASES = [
    # (code, alg, decoder kwargs, Eb/N0, frames)
    ("eg5", "fwbf", dict(block_len_p=31, k_max=100), 4.0, 1 << 15),
    ("eg5", "fwbf", dict(block_len_p=31, k_max=100), 3.0, 1 << 12),
    ("eg5", "fwbf", dict(block_len_p=93, k_max=100), 3.5, 1 << 13),
    ("eg5", "imwbf", dict(k_max=100, weight_mode="mwbf", alpha=0.0), 4.0, 1 << 11),
    ("eg5", "mlp", dict(lam=10, k_max=100), 4.0, 1 << 13),
    ("eg6", "fwbf", dict(block_len_p=128, k_max=100), 4.5, 1 << 11),
    ("gal504", "fwbf", dict(block_len_p=24, k_max=50), 4.0, 10000),
    ("qc4x32", "fwbf", dict(block_len_p=256, k_max=50), 5.0, 1 << 8),
    # explicit / QC codes with 32 | p take the fused metric + block-argmax pass
    ("gal504", "fwbf", dict(block_len_p=32, k_max=50), 3.5, 4096),
    ("gal504", "fwbf", dict(block_len_p=64, k_max=50, stall_policy="terminate"), 3.0, 4096),
    ("qc4x32", "fwbf", dict(block_len_p=32, k_max=30), 4.5, 1 << 7),
]


def _cmp(res, z, its, fl, ft, tag):
    gz = res.z()
    git = res.iterations.cpu().numpy()
    gfl = res.flags.cpu().numpy() & 3
    gft = res.flips_total.cpu().numpy()
    bad = np.nonzero((git != its) | (gfl != fl) | (gft != ft) | np.any(gz != z, axis=1))[0]
    assert bad.size == 0, f"{tag}: {bad.size} frames differ, first {bad[:8]}"


@pytest.mark.parametrize("code,alg,kw,ebn0,frames", CASES)
def test_scale_parity_vs_c_oracle(cuda_device, code, alg, kw, ebn0, frames):
    import torch
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    g = torch.Generator(device="cuda").manual_seed(hash((code, ebn0, frames)) & 0xffffffff)
    y = (1.0 + sigma * torch.randn((frames, h.n_cols), generator=g, device="cuda")).float()
    cfg = DecoderConfig(**kw)
    res = decode_batch(h, y, cfg, alg)
    p = kw.get("block_len_p")
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy(), algorithm=alg, alpha=cfg.alpha,
                                             k_max=cfg.k_max, lam=cfg.lam, p=p,
                                             weight_mode=cfg.weight_mode, stall=cfg.stall_policy,
                                             mlp_threshold=cfg.mlp_threshold)
    _cmp(res, z, its, fl, ft, f"{code}/{alg}/{ebn0}")


# -- at-scale parity of every config in the driver-run suite ----
# C (the W = 64 filtered MODE 2 kernel, widest error bound) at p in {64, 128,
# 256} x {3.5, 4.0, 4.5} dB; B at p in {31, 93} over the whole 3.0-5.0 dB
# sweep; D at its config point.  Every frame is compared with the C oracle.
SWEEP = ([("eg6", p, db, 1 << 12, 100) for p in (64, 128, 256) for db in (3.5, 4.0, 4.5)] +
         [("eg5", p, db, 1 << 14, 100) for p in (31, 93) for db in (3.0, 3.5, 4.0, 4.5, 5.0)] +
         [("qc4x32", 256, 5.0, 1 << 12, 50)])


def _oracle_threads():
    import os
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())


@pytest.mark.parametrize("code,p,ebn0,frames,kmax", SWEEP)
def test_sweep_parity_vs_c_oracle(cuda_device, code, p, ebn0, frames, kmax):
    import torch
    from paper_1206_3362_b200 import device_code
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    g = torch.Generator(device="cuda").manual_seed(int(ebn0 * 10) * 1000 + p)
    # rows padded to a 16-byte multiple (ld = 1024 / 4096): the circulant
    # kernels then stage each frame's row with a TMA bulk copy one frame ahead
    ld = (h.n_cols + 3) // 4 * 4
    ybuf = torch.zeros((frames, ld), dtype=torch.float32, device="cuda")
    y = ybuf[:, :h.n_cols]
    y.copy_(1.0 + sigma * torch.randn((frames, h.n_cols), generator=g, device="cuda"))
    cfg = DecoderConfig(block_len_p=p, k_max=kmax)
    dc = device_code(h, 0)
    dc.filter_stats(reset=True)
    res = decode_batch(h, y, cfg, "fwbf")
    torch.cuda.synchronize()
    fs = dc.filter_stats(reset=True)
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy(), threads=_oracle_threads(), algorithm="fwbf",
                                             alpha=0.2, k_max=kmax, p=p)
    _cmp(res, z, its, fl, ft, f"{code}/p{p}/{ebn0}")
    if code == "eg6" and p == 64 and ebn0 <= 4.0:
        # the filtered metric had to resolve decisions exactly (the fallback ran)
        assert fs[0] > 0, fs


@pytest.mark.parametrize("noise", ["f32", "f64"])
def test_sweep_parity_device_noise_64k(cuda_device, noise):
    """Config E at 2^16 frames: on-device reference channel, every frame vs the C oracle."""
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    res = decode_awgn(h, cfg, "fwbf", 5, 1 << 30, 1 << 16, sigma, noise=noise, return_y=True)
    z, its, fl, ft = COracle(h).decode_batch(res.y.cpu().numpy(), threads=_oracle_threads(), algorithm="fwbf",
                                             alpha=0.2, k_max=100, p=31)
    _cmp(res, z, its, fl, ft, f"E-{noise}")
    hist = res.iter_hist.cpu().numpy()
    assert np.array_equal(hist, np.bincount(its, minlength=101))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_counters_equal_single_gpu(cuda_device, world):
    """G = 1 vs G shards (run here sequentially on one GPU,
    each shard a separate decode_awgn call over its frame_shard range).
    Per-frame results and the summed counters equal the single call's: noise
    is keyed by the global frame index."""
    import torch
    from paper_1206_3362_b200.sharding import frame_shard
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(3.5, code_rate("eg5"))
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    first, count = 1000, 30011
    one = decode_awgn(h, cfg, "fwbf", 9, first, count, sigma, noise="f32")
    parts, cnt = [], torch.zeros_like(one.counters)
    for r in range(world):
        s0, n0 = frame_shard(first, count, r, world)
        part = decode_awgn(h, cfg, "fwbf", 9, s0, n0, sigma, noise="f32")
        parts.append(part)
        cnt += part.counters
    assert torch.equal(cnt, one.counters)
    for name in ("iterations", "flags", "z_bits", "bit_errors"):
        assert torch.equal(torch.cat([getattr(q, name) for q in parts]), getattr(one, name)), name
    assert torch.equal(sum(q.iter_hist for q in parts), one.iter_hist)


@pytest.mark.parametrize("noise", ["f32", "f64"])
def test_scale_parity_device_noise(cuda_device, noise):
    """Config E path: the device draws the reference channel; the C oracle
    decodes the very same values (returned by the kernel)."""
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    res = decode_awgn(h, cfg, "fwbf", 11, 1 << 20, 1 << 13, sigma, noise=noise, return_y=True)
    z, its, fl, ft = COracle(h).decode_batch(res.y.cpu().numpy(), algorithm="fwbf", alpha=0.2,
                                             k_max=100, p=31)
    _cmp(res, z, its, fl, ft, f"awgn-{noise}")


@pytest.mark.parametrize("code,p,stall,dtype", [
    ("gal504", 32, "flip-global-max", "f32"), ("gal504", 96, "terminate", "f32"),
    ("gal504", 64, "flip-global-max", "f64"), ("qc4x32", 256, "flip-global-max", "f32"),
    ("qc4x32", 512, "terminate", "f64")])
def test_fused_pass_matches_unfused(cuda_device, monkeypatch, code, p, stall, dtype):
    """The fused metric + block-argmax pass (explicit/QC, 32 | p) gives the same
    flip sequence as the metric-buffer path, frame by frame."""
    h = build_code(code)
    n = h.n_cols
    rng = np.random.default_rng(p)
    sigma = 0.62 if code == "gal504" else 0.45
    y = (1.0 + sigma * rng.standard_normal((256, n))).astype(np.float32 if dtype == "f32" else np.float64)
    cfg = DecoderConfig(block_len_p=p, k_max=40, stall_policy=stall)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    monkeypatch.setenv("FWBF_NO_FUSED", "1")
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    assert np.array_equal(a.iterations.cpu().numpy(), b.iterations.cpu().numpy())
    assert np.array_equal(a.flags.cpu().numpy(), b.flags.cpu().numpy())
    assert a.flip_logs() == b.flip_logs()


@pytest.mark.parametrize("code,weight_mode,alpha,ebn0", [
    ("eg4", "imwbf", 0.2, 3.0), ("eg5", "imwbf", 0.2, 4.0), ("eg5", "mwbf", 0.0, 4.0),
    ("eg6", "imwbf", 0.3, 4.0)])
def test_imwbf_incremental_matches_full_recompute(cuda_device, monkeypatch, code, weight_mode, alpha, ebn0):
    """IMWBF on the split path keeps the metric incrementally (integer limb
    updates per toggled check); it must give the flip sequence of the full
    per-iteration recomputation, frame by frame, and the oracle's."""
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    rng = np.random.default_rng(11)
    frames = 512 if h.n_cols < 4000 else 128
    y = (1.0 + sigma * rng.standard_normal((frames, h.n_cols))).astype(np.float32)
    cfg = DecoderConfig(alpha=alpha, k_max=60, weight_mode=weight_mode)
    a = decode_batch(h, y, cfg, "imwbf", flip_log=True)
    monkeypatch.setenv("FWBF_NO_INC", "1")
    b = decode_batch(h, y, cfg, "imwbf", flip_log=True)
    assert np.array_equal(a.iterations.cpu().numpy(), b.iterations.cpu().numpy())
    assert np.array_equal(a.z(), b.z())
    assert a.flip_logs() == b.flip_logs()
    z, its, fl, ft = COracle(h).decode_batch(y[:64], algorithm="imwbf", alpha=alpha, k_max=60,
                                             weight_mode=weight_mode)
    assert np.array_equal(a.iterations.cpu().numpy()[:64], its)
    assert np.array_equal(a.z()[:64], z)


def test_deterministic_across_runs(cuda_device):
    """Frames are claimed from an atomic queue in a different order every run;
    the per-frame results and the counters must not depend on it."""
    import torch
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(3.5, code_rate("eg5"))
    g = torch.Generator(device="cuda").manual_seed(123)
    y = (1.0 + sigma * torch.randn((1 << 17, h.n_cols), generator=g, device="cuda")).float()
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    a = decode_batch(h, y, cfg, "fwbf")
    b = decode_batch(h, y, cfg, "fwbf")
    for name in ("z_bits", "iterations", "flags", "flips_total", "counters"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
