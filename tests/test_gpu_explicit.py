"""The one-frame-per-warp FWBF kernel for small explicit codes (fwbf_explicit.cu):
bit-exact against the C oracle and against the CTA-per-frame kernel
(FWBF_NO_WARP=1) -- hard decisions, iterations, flags, flip logs, counters --
over block lengths (groups of 1..32 lanes per block), stall policies, weight
modes, float4 and scalar row loads, and a dv = 4 code."""

import numpy as np
import pytest

from oracle import wbf_oracle as O
from oracle.c_oracle import COracle
from paper_1206_3362_b200 import DecoderConfig, ParityCheckMatrix, decode_batch, gallager_rc
from tests.golden.codebook import build_code, code_rate

pytestmark = pytest.mark.gpu


def _y(h, frames, ebn0, rate, seed, pad):
    import torch
    n = h.n_cols
    sigma = O.ebn0_to_sigma(ebn0, rate)
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld = (n + 3) // 4 * 4 + (4 if pad else 0)
    buf = torch.zeros((frames, ld if pad else n), dtype=torch.float32, device="cuda")
    y = buf[:, :n]
    y.copy_(1.0 + sigma * torch.randn((frames, n), generator=g, device="cuda"))
    return y


def _same(a, b):
    import torch
    for name in ("z_bits", "iterations", "flags", "flips_total", "bit_errors", "counters", "iter_hist"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name


@pytest.fixture(autouse=True, params=["xinc", "xdecode"])
def warp_kernel_variant(request, monkeypatch):
    """The warp-kernel cases run on both one-frame-per-warp kernels: the
    incremental one (stored float32 roundings of the exact metrics, only the
    columns of toggled checks recomputed; the default) and the full-pass one
    (FWBF_NO_XINC=1).  The QC cases below ignore the switch."""
    if request.param == "xdecode":
        monkeypatch.setenv("FWBF_NO_XINC", "1")
    return request.param


@pytest.mark.parametrize("p", [1, 3, 7, 24, 32, 63, 96, 252, 504, 1000])
@pytest.mark.parametrize("stall", ["flip-global-max", "terminate"])
def test_warp_kernel_matches_cta_kernel_and_oracle(cuda_device, monkeypatch, warp_kernel_variant, p, stall):
    from paper_1206_3362_b200 import _native as nat
    h = build_code("gal504")
    y = _y(h, 3000, 3.5, code_rate("gal504"), p, pad=(p % 2 == 0))
    y[7] = (y[7] * 4).round() / 4                     # equal metrics: exact rounds / exact stall argmax
    y[8] = 0.0
    cfg = DecoderConfig(block_len_p=p, k_max=50, stall_policy=stall)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    assert nat.last_kernel() == warp_kernel_variant
    monkeypatch.setenv("FWBF_NO_WARP", "1")
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    _same(a, b)
    assert a.flip_logs() == b.flip_logs()
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy(), algorithm="fwbf", alpha=0.2, k_max=50, p=p,
                                             stall=stall)
    assert np.array_equal(a.iterations.cpu().numpy(), its)
    assert np.array_equal(a.z(), z)
    assert np.array_equal(a.flips_total.cpu().numpy(), ft)


@pytest.mark.parametrize("weight_mode,alpha", [("mwbf", 0.0), ("mwbf", 0.3), ("imwbf", 1.0), ("imwbf", 0.0)])
def test_warp_kernel_weight_modes(cuda_device, weight_mode, alpha):
    h = build_code("gal504")
    y = _y(h, 512, 4.0, code_rate("gal504"), 7, pad=True)
    cfg = DecoderConfig(block_len_p=24, k_max=40, alpha=alpha, weight_mode=weight_mode)
    res = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    logs = res.flip_logs()
    g = O.Graph.of(h)
    yy = y.cpu().numpy()
    for i in range(0, 512, 16):
        r = O.decode(g, yy[i], "fwbf", alpha=alpha, k_max=40, p=24, weight_mode=weight_mode)
        assert int(res.iterations[i]) == r.iterations and logs[i] == r.flip_log, i


def test_warp_kernel_dv4_and_columns_without_checks(cuda_device):
    """A (4, 8)-regular code, and an irregular code whose last columns belong to
    no check (metric = -alpha|y|)."""
    h = gallager_rc(512, 4, 8, seed=3)
    y = _y(h, 2000, 4.0, 0.5, 1, pad=True)
    cfg = DecoderConfig(block_len_p=16, k_max=30)
    res = decode_batch(h, y, cfg, "fwbf")
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy(), algorithm="fwbf", alpha=0.2, k_max=30, p=16)
    assert np.array_equal(res.iterations.cpu().numpy(), its) and np.array_equal(res.z(), z)
    rng = np.random.default_rng(4)
    rows = [np.sort(rng.choice(90, size=5, replace=False)) for _ in range(50)]
    h2 = ParityCheckMatrix(rows, 100)                  # columns 90..99 are in no check
    y2 = (1.0 + 0.7 * rng.standard_normal((300, 100))).astype(np.float32)
    y2[:, 95] = -0.5                                   # a hard error no check can see
    for p in (5, 10, 100):
        cfg = DecoderConfig(block_len_p=p, k_max=20, alpha=0.5)
        res = decode_batch(h2, y2, cfg, "fwbf", flip_log=True)
        logs = res.flip_logs()
        g = O.Graph.of(h2)
        for i in range(0, 300, 7):
            r = O.decode(g, y2[i], "fwbf", alpha=0.5, k_max=20, p=p)
            assert int(res.iterations[i]) == r.iterations and logs[i] == r.flip_log, (p, i)


def test_warp_kernels_agree_on_special_frames(cuda_device, monkeypatch, warp_kernel_variant):
    """Non-finite, all-zero and heavily quantised frames: both warp kernels
    give what the CTA kernel gives (the incremental one decides such frames on
    exact values everywhere)."""
    import torch
    h = build_code("gal504")
    y = _y(h, 400, 4.0, code_rate("gal504"), 77, pad=True)
    y[3, 5] = float("nan")
    y[4, 100] = float("inf")
    y[5, 200] = float("-inf")
    y[6] = 0.0
    y[10:200] = torch.round(y[10:200] * 2) / 2
    for p, stall in ((24, "flip-global-max"), (24, "terminate"), (63, "flip-global-max")):
        cfg = DecoderConfig(block_len_p=p, k_max=40, stall_policy=stall, alpha=0.5)
        a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
        monkeypatch.setenv("FWBF_NO_WARP", "1")
        b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
        monkeypatch.delenv("FWBF_NO_WARP")
        _same(a, b)
        assert a.flip_logs() == b.flip_logs()


# ---- quasi-cyclic kernel (fwbf_qc.cu): config D's path ----

def _qc_code(seed, jb, kb, z, absent):
    from paper_1206_3362_b200.codes import qc_from_shifts
    rng = np.random.default_rng(seed)
    sh = rng.integers(0, z, size=(jb, kb))
    if absent:
        sh[rng.random((jb, kb)) < 0.2] = -1
        sh[0, :] = np.maximum(sh[0, :], 0)        # every column keeps a check
    return qc_from_shifts(sh, z)


@pytest.mark.parametrize("code,p,stall,wmode", [
    ("qc4x32", 256, "flip-global-max", "imwbf"), ("qc4x32", 512, "terminate", "imwbf"),
    ("qc4x32", 32, "flip-global-max", "mwbf"), ("r3x16z64", 64, "flip-global-max", "imwbf"),
    ("r4x12z32a", 32, "terminate", "imwbf"), ("r2x8z128a", 128, "flip-global-max", "imwbf"),
    ("r4x20z16a", 16 * 2, "flip-global-max", "mwbf")])
def test_qc_kernel_matches_cta_kernel_and_oracle(cuda_device, monkeypatch, code, p, stall, wmode):
    if code == "qc4x32":
        h = build_code(code)
    else:
        jb, rest = code[1:].split("x")
        kb, zz = rest.split("z")
        h = _qc_code(len(code) + p, int(jb), int(kb), int(zz.rstrip("a")), zz.endswith("a"))
    frames = 256 if h.n_cols > 4000 else 2000
    y = _y(h, frames, 5.0 if h.n_cols > 4000 else 3.5, 0.8 if h.n_cols > 4000 else 0.6, p, pad=True)
    cfg = DecoderConfig(block_len_p=p, k_max=30, stall_policy=stall, weight_mode=wmode)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    monkeypatch.setenv("FWBF_NO_QCK", "1")
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    _same(a, b)
    assert a.flip_logs() == b.flip_logs()
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy()[:128], algorithm="fwbf", alpha=0.2, k_max=30, p=p,
                                             stall=stall, weight_mode=wmode)
    assert np.array_equal(a.iterations.cpu().numpy()[:128], its)
    assert np.array_equal(a.z()[:128], z)


@pytest.mark.parametrize("quant", [0.25, 0.5])
@pytest.mark.parametrize("p,alpha", [(256, 0.2), (64, 1.0), (512, 0.0)])
def test_qc_kernel_quantised_ties(cuda_device, monkeypatch, quant, p, alpha):
    """Quantised y: many exact ties between metrics, and metrics that are +0.0
    in the reference but -0.0 in a sum started at its first term -- the
    REDUX block argmax must key them equally (lowest index wins)."""
    import torch
    h = build_code("qc4x32")
    y = _y(h, 384, 5.0, 0.875, 11 + p, pad=True)
    y.copy_(torch.round(y / quant) * quant)
    cfg = DecoderConfig(block_len_p=p, k_max=25, alpha=alpha)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    monkeypatch.setenv("FWBF_NO_QCK", "1")
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    _same(a, b)
    assert a.flip_logs() == b.flip_logs()
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy()[:96], algorithm="fwbf", alpha=alpha, k_max=25, p=p)
    assert np.array_equal(a.iterations.cpu().numpy()[:96], its)
    assert np.array_equal(a.z()[:96], z)


# ---- incremental quasi-cyclic kernel (qinc_kernel): stored metric keys, only
# the columns of toggled checks recomputed ----

@pytest.mark.parametrize("code,p,stall", [
    ("qc4x32", 256, "flip-global-max"), ("r2x40z32", 32, "flip-global-max"),
    ("r3x36z64a", 64, "terminate"), ("r4x12z32a", 32, "flip-global-max")])
def test_qc_incremental_kernel_equals_full_pass(cuda_device, monkeypatch, code, p, stall):
    """The incremental kernel against the full-pass QC kernel (FWBF_NO_QCINC)
    and the oracle, on batches that also hold frames it must decide exactly
    everywhere (non-finite y), all-zero frames and quantised frames (equal
    keys); codes wider than 32 block columns take the second update loop."""
    import torch
    from paper_1206_3362_b200 import _native as nat
    if code == "qc4x32":
        h = build_code(code)
    else:
        jb, rest = code[1:].split("x")
        kb, zz = rest.split("z")
        h = _qc_code(len(code) + p, int(jb), int(kb), int(zz.rstrip("a")), zz.endswith("a"))
    big = h.n_cols > 4000
    frames = 192 if big else 1500
    y = _y(h, frames, 5.0 if big else 3.5, 0.8 if big else 0.6, 3 * p + 1, pad=True)
    y[5, 7] = float("nan")
    y[6, 11] = float("inf")
    y[7, 3] = float("-inf")
    y[8, :] = 0.0
    y[9:40] = torch.round(y[9:40] * 2) / 2                 # many equal metrics
    cfg = DecoderConfig(block_len_p=p, k_max=30, stall_policy=stall, alpha=0.3)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    assert nat.last_kernel() == "qinc"
    monkeypatch.setenv("FWBF_NO_QCINC", "1")
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    assert nat.last_kernel() == "qdecode"
    _same(a, b)
    assert a.flip_logs() == b.flip_logs()
    sel = [i for i in range(64) if i not in (5, 6, 7)]    # finite frames against the oracle
    z, its, fl, ft = COracle(h).decode_batch(y.cpu().numpy()[sel], algorithm="fwbf", alpha=0.3, k_max=30, p=p,
                                             stall=stall)
    assert np.array_equal(a.iterations.cpu().numpy()[sel], its)
    assert np.array_equal(a.z()[sel], z)
