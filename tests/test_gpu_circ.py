"""The filtered kernel for cyclic EG codes (csrc/fwbf_circ.cu): FWBF and MLP-WBF.

It decodes every frame its guard admits (finite y, some |y| > 0, the fp64
guard of DESIGN.md section 2) and defers the rest to decode_kernel through a
frame list.  Its results must equal decode_kernel's MODE 2 (FWBF_NO_CDEC=1)
and the oracle bit for bit: hard decisions, iterations, flags, flip counts
and the flip sequence, for compiled-in and runtime block lengths, both stall
policies, and batches that mix deferred frames in.  MLP-WBF (lambda <= 31)
runs on the same kernel with a filtered top-lambda selection and must equal
decode_kernel's exact MODE 0 and the oracle.  Round 2, fourth session: the
gather reads the minima quantised to 16 bits on a per-frame grid (Q16); the
float32 gather remains as FWBF_Q16=0, and every case here runs on both.
"""

import os

import numpy as np
import pytest

from oracle import wbf_oracle as O
from oracle.c_oracle import COracle
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from tests.golden.codebook import build_code, code_rate

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["q16", "f32"])
def gather_variant(request, monkeypatch):
    """Every case runs on both gathers of the kernel: the 16-bit quantised one
    (the default) and the float32 one (FWBF_Q16=0); both must give the
    reference's results bit for bit -- only the width of the filter band, and
    so the number of exact re-decisions, differs."""
    monkeypatch.setenv("FWBF_Q16", "1" if request.param == "q16" else "0")
    return request.param


def _frames(code, ebn0, frames, seed, quant=None):
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    rng = np.random.default_rng(seed)
    y = 1.0 + sigma * rng.standard_normal((frames, h.n_cols))
    if quant:
        y = np.round(y * quant) / quant
    return h, y.astype(np.float32)


def _decode(h, y, cfg, cdec=True, alg="fwbf"):
    """decode_batch with or without the circulant kernel (FWBF_NO_CDEC is read per launch)."""
    if cdec:
        os.environ.pop("FWBF_NO_CDEC", None)
    else:
        os.environ["FWBF_NO_CDEC"] = "1"
    try:
        r = decode_batch(h, y, cfg, alg, flip_log=True)
        kern = nat.last_kernel()
    finally:
        os.environ.pop("FWBF_NO_CDEC", None)
    return r, kern


def _same(a, b, tag, flag_mask=0xff):
    """flag_mask 11 (converged, stalled, non-finite): the metric-path bits may
    differ from decode_kernel's exact MODE 0 (it flags frames that fail the
    split-fp32 guard as fp64-guarded; the filtered kernel's path is one)."""
    for name in ("iterations", "flips_total", "flags"):
        u, v = getattr(a, name).cpu().numpy(), getattr(b, name).cpu().numpy()
        if name == "flags":
            u, v = u & flag_mask, v & flag_mask
        assert np.array_equal(u, v), f"{tag}: {name} differs at {np.nonzero(u != v)[0][:8]}"
    assert np.array_equal(a.z_bits.cpu().numpy(), b.z_bits.cpu().numpy()), f"{tag}: z differs"
    assert a.flip_logs() == b.flip_logs(), f"{tag}: flip logs differ"


def _vs_oracle(res, h, y, cfg, tag, rows=None, alg="fwbf"):
    rows = np.arange(y.shape[0]) if rows is None else rows
    z, its, fl, ft = COracle(h).decode_batch(y[rows], algorithm=alg, alpha=cfg.alpha, k_max=cfg.k_max,
                                             lam=cfg.lam, p=cfg.block_len_p, weight_mode=cfg.weight_mode,
                                             stall=cfg.stall_policy, mlp_threshold=cfg.mlp_threshold)
    bad = np.nonzero((res.iterations.cpu().numpy()[rows] != its) | ((res.flags.cpu().numpy()[rows] & 3) != fl) |
                     (res.flips_total.cpu().numpy()[rows] != ft) | np.any(res.z()[rows] != z, axis=1))[0]
    assert bad.size == 0, f"{tag}: {bad.size} frames differ from the oracle, first {rows[bad[:8]]}"


@pytest.mark.parametrize("code,p,ebn0,frames", [
    ("eg5", 31, 4.0, 2048),     # the headline shape (block length compiled in)
    ("eg5", 31, 3.0, 512),
    ("eg5", 93, 4.0, 1024),     # compiled in, p > 32
    ("eg5", 16, 4.0, 512),      # runtime p, the smallest the kernel takes
    ("eg5", 32, 4.5, 512),
    ("eg5", 100, 3.5, 512),     # runtime p > 32, ragged last block
    ("eg5", 1023, 4.0, 256),    # one block
    ("eg4", 17, 3.5, 1024),     # EG(255), W = 16
    ("eg4", 51, 4.0, 1024),
    ("eg6", 64, 4.0, 128),      # EG(4095), W = 64, compiled in
    ("eg6", 256, 3.5, 96),
    ("eg6", 100, 4.5, 96),      # EG(4095), runtime p
])
def test_circ_kernel_equals_mode2_and_oracle(cuda_device, code, p, ebn0, frames):
    h, y = _frames(code, ebn0, frames, seed=p * 131 + frames)
    cfg = DecoderConfig(block_len_p=p, k_max=60, alpha=0.2)
    a, ka = _decode(h, y, cfg, True)
    b, kb = _decode(h, y, cfg, False)
    assert ka == "cdecode+decode_kernel" and kb == "decode_kernel", (ka, kb)
    _same(a, b, f"{code}/p{p}/{ebn0}dB")
    _vs_oracle(a, h, y, cfg, f"{code}/p{p}/{ebn0}dB", rows=np.arange(min(frames, 256)))


@pytest.mark.parametrize("stall,alpha,quant", [
    ("flip-global-max", 1.5, 16),   # maxima near / below 0: stalls and exact fallbacks
    ("terminate", 1.5, 8),
    ("flip-global-max", 0.2, 4),    # coarse quantisation: many exact ties
])
def test_circ_kernel_stalls_and_ties(cuda_device, stall, alpha, quant):
    h, y = _frames("eg5", 3.5, 256, seed=7 + quant, quant=quant)
    cfg = DecoderConfig(block_len_p=31, k_max=40, alpha=alpha, stall_policy=stall)
    a, ka = _decode(h, y, cfg, True)
    b, _ = _decode(h, y, cfg, False)
    assert ka == "cdecode+decode_kernel"
    _same(a, b, f"{stall}/a{alpha}/q{quant}")
    _vs_oracle(a, h, y, cfg, f"{stall}/a{alpha}/q{quant}")


def test_circ_kernel_defers_unguarded_frames(cuda_device):
    """Frames the filtered guard rejects go to decode_kernel through the defer
    list, interleaved with ordinary frames; every frame's result is the one
    decode_kernel alone produces (and the oracle's for the finite ones)."""
    h, y = _frames("eg5", 4.0, 640, seed=99)
    special = {}
    special[3] = np.zeros(h.n_cols, np.float32)                    # all |y| == 0
    v = y[10].copy(); v[5] = np.inf; special[10] = v                 # non-finite
    v = y[11].copy(); v[700] = np.nan; special[11] = v
    v = y[200].copy(); v[17] = 3e37; v[18] = 1e-38; special[200] = v  # beyond the fp64 guard
    v = y[201].copy(); v[::7] = -0.0; special[201] = v               # signed zeros (guard passes)
    v = y[333].copy(); v[::3] = 1e-30; special[333] = v              # huge range
    for i, v in special.items():
        y[i] = v
    cfg = DecoderConfig(block_len_p=31, k_max=50, alpha=0.2)
    a, ka = _decode(h, y, cfg, True)
    b, _ = _decode(h, y, cfg, False)
    assert ka == "cdecode+decode_kernel"
    _same(a, b, "mixed batch")
    finite = np.array([i for i in range(y.shape[0]) if np.all(np.isfinite(y[i]))])
    _vs_oracle(a, h, y, cfg, "mixed batch", rows=finite[finite < 400])


def test_circ_kernel_coarse_quantisation_grid(cuda_device):
    """Frames whose largest check minimum is far above the others (every
    column of one check, or of many, scaled up): the 16-bit grid is then
    coarse for all the other minima, most block decisions fall inside the
    widened band and are re-decided exactly -- results must not change."""
    from paper_1206_3362_b200 import device_code
    h, y = _frames("eg5", 4.0, 384, seed=41)
    rows = h.row_adj
    for i in range(0, 128):                       # one check's 32 columns x 2^10
        y[i, list(rows[(7 * i) % h.n_rows])] *= np.float32(1024.0)
    for i in range(128, 256):                     # a third of the columns x 2^6 (many large minima)
        y[i, ::3] *= np.float32(64.0)
    for i in range(256, 320):                     # tiny values next to ordinary ones
        y[i, 1::2] *= np.float32(2.0 ** -12)
    for i in range(320, 352):                     # a zero in every check: every minimum is 0 (vmax = 0)
        y[i, ::2] = 0.0
    for i in range(352, 384):                     # ... and in most checks
        y[i, ::5] = 0.0
    for mlp in (False, True):
        cfg = DecoderConfig(lam=7, k_max=40) if mlp else DecoderConfig(block_len_p=31, k_max=60, alpha=0.2)
        alg = "mlp" if mlp else "fwbf"
        dc = device_code(h)
        dc.filter_stats(reset=True)
        a, ka = _decode(h, y, cfg, True, alg=alg)
        st = dc.filter_stats(reset=True)
        b, _ = _decode(h, y, cfg, False, alg=alg)
        assert ka == "cdecode+decode_kernel"
        _same(a, b, f"coarse grid {alg}", flag_mask=11 if mlp else 0xff)
        _vs_oracle(a, h, y, cfg, f"coarse grid {alg}", alg=alg)
        assert mlp or st[0] > 0                   # the exact path ran


def test_circ_kernel_staged_rows(cuda_device):
    """TMA-staged input rows (16-byte row stride, forced for a small batch)
    give the same results as element loads."""
    import torch
    h, y = _frames("eg5", 4.0, 300, seed=5)
    cfg = DecoderConfig(block_len_p=31, k_max=60)
    ypad = torch.zeros((y.shape[0], 1024), dtype=torch.float32, device="cuda:0")
    ypad[:, :h.n_cols] = torch.from_numpy(y).cuda()
    os.environ["FWBF_FORCE_YSTAGE"] = "1"
    try:
        a = decode_batch(h, ypad[:, :h.n_cols], cfg, "fwbf", flip_log=True)
        assert nat.last_kernel() == "cdecode+decode_kernel"
    finally:
        os.environ.pop("FWBF_FORCE_YSTAGE", None)
    b, _ = _decode(h, y, cfg, False)
    _same(a, b, "staged rows")


@pytest.mark.parametrize("code,lam,ebn0,thr,stall,quant,frames", [
    ("eg5", 10, 4.0, True, "flip-global-max", None, 2048),   # config E's comparison decoder
    ("eg5", 10, 3.0, True, "flip-global-max", None, 512),
    ("eg5", 1, 4.0, True, "flip-global-max", None, 512),
    ("eg5", 3, 3.5, False, "flip-global-max", None, 512),    # unthresholded: lambda flips every iteration
    ("eg5", 31, 4.0, True, "flip-global-max", None, 512),    # the largest lambda the kernel takes
    ("eg5", 10, 3.5, True, "terminate", None, 512),
    ("eg5", 10, 3.5, True, "flip-global-max", 8, 512),       # quantised: ties, exact decisions
    ("eg5", 5, 3.5, True, "terminate", 4, 512),
    ("eg4", 10, 4.0, True, "flip-global-max", None, 1024),   # EG(255)
    ("eg6", 10, 4.0, True, "flip-global-max", None, 96),     # EG(4095)
])
def test_circ_kernel_mlp_equals_mode0_and_oracle(cuda_device, code, lam, ebn0, thr, stall, quant, frames):
    h, y = _frames(code, ebn0, frames, seed=lam * 17 + frames, quant=quant)
    cfg = DecoderConfig(lam=lam, k_max=40, alpha=1.5 if quant else 0.2, mlp_threshold=thr, stall_policy=stall)
    a, ka = _decode(h, y, cfg, True, "mlp")
    b, kb = _decode(h, y, cfg, False, "mlp")
    assert ka == "cdecode+decode_kernel" and kb == "decode_kernel", (ka, kb)
    _same(a, b, f"mlp/{code}/l{lam}/{ebn0}dB/q{quant}", flag_mask=11)
    _vs_oracle(a, h, y, cfg, f"mlp/{code}/l{lam}", rows=np.arange(min(frames, 256)), alg="mlp")
