"""The filtered FWBF metric ("filtered"): on split-path
frames the gather sums the signed check minima directly in fp32 and every
block decision closer than the per-frame error bound is re-decided with exact
column sums.  Results must equal the exact path and the oracle bit for bit;
these cases force the exact fallback (ties from quantised y, metrics near 0,
stalls, a huge dynamic range that widens the bound) and check it ran.
"""

import numpy as np
import pytest

from oracle import wbf_oracle as O
from oracle.c_oracle import COracle
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.decoders import device_code
from tests.golden.codebook import build_code, code_rate

pytestmark = pytest.mark.gpu

NOFILTER = 4


def _frames(code, ebn0, frames, seed, quant=None):
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    rng = np.random.default_rng(seed)
    y = 1.0 + sigma * rng.standard_normal((frames, h.n_cols))
    if quant:
        y = np.round(y * quant) / quant        # many exactly equal metrics
    return h, y.astype(np.float32)


def _same(a, b, tag):
    for name in ("iterations", "flips_total"):
        u, v = getattr(a, name).cpu().numpy(), getattr(b, name).cpu().numpy()
        assert np.array_equal(u, v), f"{tag}: {name} differs at {np.nonzero(u != v)[0][:8]}"
    assert np.array_equal(a.z_bits.cpu().numpy(), b.z_bits.cpu().numpy()), f"{tag}: z differs"
    # converged / stalled / non-finite must agree; the metric path bits may
    # not (the filtered kernels run frames that fail the split-fp32 guard on
    # the ordered path instead of the guarded fp64 one)
    fa, fb = a.flags.cpu().numpy(), b.flags.cpu().numpy()
    assert np.array_equal(fa & 11, fb & 11), f"{tag}: flags differ"


def _oracle(h, y, cfg):
    return COracle(h).decode_batch(y, algorithm="fwbf", alpha=cfg.alpha, k_max=cfg.k_max, lam=cfg.lam,
                                   p=cfg.block_len_p, weight_mode=cfg.weight_mode,
                                   stall=cfg.stall_policy, mlp_threshold=cfg.mlp_threshold)


def _vs_oracle(res, h, y, cfg, tag):
    z, its, fl, ft = _oracle(h, y, cfg)
    bad = np.nonzero((res.iterations.cpu().numpy() != its) | ((res.flags.cpu().numpy() & 3) != fl) |
                     (res.flips_total.cpu().numpy() != ft) | np.any(res.z() != z, axis=1))[0]
    assert bad.size == 0, f"{tag}: {bad.size} frames differ from the oracle, first {bad[:8]}"


@pytest.mark.parametrize("code,p,quant,alpha,stall", [
    ("eg5", 31, 8, 0.2, "flip-global-max"),
    ("eg5", 93, 4, 0.2, "flip-global-max"),
    ("eg5", 1023, 8, 0.2, "flip-global-max"),     # one block: the stall argmax path
    ("eg5", 31, 16, 1.5, "flip-global-max"),      # large alpha: maxima near / below 0
    ("eg5", 31, 8, 1.5, "terminate"),
    ("eg4", 15, 4, 0.2, "flip-global-max"),
    ("eg6", 64, 8, 0.2, "flip-global-max"),       # W = 64
])
def test_quantised_ties_resolved_exactly(cuda_device, code, p, quant, alpha, stall):
    h, y = _frames(code, 3.5, 96 if code != "eg6" else 32, seed=p * 7 + quant, quant=quant)
    cfg = DecoderConfig(block_len_p=p, k_max=40, alpha=alpha, stall_policy=stall)
    dc = device_code(h)
    dc.filter_stats(reset=True)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    st = dc.filter_stats(reset=True)
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True, force_ordered=NOFILTER)
    _same(a, b, f"{code}/p{p}/q{quant}")
    assert a.flip_logs() == b.flip_logs()
    _vs_oracle(a, h, y, cfg, f"{code}/p{p}/q{quant}")
    split = (a.flags.cpu().numpy() & 16) != 0
    if split.any():
        assert st[0] > 0, "quantised inputs should force exact block resolutions"
    if p == 1023 and split.any():
        assert st[1] >= 0


def test_stall_argmax_resolved_exactly(cuda_device):
    # p = 1 makes every column its own block, so a stall (no positive metric)
    # takes the global argmax over N approximate block values; quantised y
    # gives exact ties among them
    h, y = _frames("eg5", 3.0, 64, seed=5, quant=4)
    cfg = DecoderConfig(block_len_p=1, k_max=30, alpha=3.0)
    dc = device_code(h)
    dc.filter_stats(reset=True)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    st = dc.filter_stats(reset=True)
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True, force_ordered=NOFILTER)
    _same(a, b, "stall")
    assert a.flip_logs() == b.flip_logs()
    _vs_oracle(a, h, y, cfg, "stall")
    if ((a.flags.cpu().numpy() & 16) != 0).any() and (a.flags.cpu().numpy() & 2).any():
        assert st[1] > 0, "stalls on quantised inputs should need an exact global argmax"


def test_wide_bound_frames(cuda_device):
    # one huge |y| per frame makes the filter's bound (which scales with the
    # largest check minimum) wide, so many decisions fall back; still exact
    h, y = _frames("eg5", 4.0, 64, seed=9)
    y[:, 7] = 3.0e3
    y[::2, 500] = -2.5e3
    cfg = DecoderConfig(block_len_p=31, k_max=60)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True, force_ordered=NOFILTER)
    _same(a, b, "wide")
    _vs_oracle(a, h, y, cfg, "wide")


@pytest.mark.parametrize("ebn0,p", [(4.0, 31), (3.0, 93), (5.0, 31)])
def test_filter_equals_exact_full_size(cuda_device, ebn0, p):
    import torch
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(ebn0, code_rate("eg5"))
    g = torch.Generator(device="cuda").manual_seed(int(ebn0 * 10) + p)
    y = (1.0 + sigma * torch.randn((1 << 16, 1023), generator=g, device="cuda")).float()
    cfg = DecoderConfig(block_len_p=p, k_max=100)
    a = decode_batch(h, y, cfg, "fwbf")
    b = decode_batch(h, y, cfg, "fwbf", force_ordered=NOFILTER)
    _same(a, b, f"full/{ebn0}/{p}")
    ca, cb = a.counters.cpu().numpy(), b.counters.cpu().numpy()
    keep = [i for i in range(len(ca)) if i != nat.CNT_ORDERED_FRAMES]
    assert np.array_equal(ca[keep], cb[keep])


@pytest.mark.parametrize("tiny", [3e-7, 1e-12, 1e-30])
def test_fp64_guarded_frames_take_the_filtered_path(cuda_device, tiny):
    # One tiny |y| per frame makes the quantum q tiny: the split-fp32 guard
    # fails but the fp64 guard holds, so the MODE 2 kernel filters these frames
    # too (its exact fallback only needs the fp64 guard); 1e-30 also leaves the
    # quantum range of the coarse corrections, which sends frames to the
    # ordered path.  Results must equal the oracle either way.
    h, y = _frames("eg5", 3.5, 64, seed=21)
    y[:, 100] = tiny
    y[1::2, 600] = -tiny
    cfg = DecoderConfig(block_len_p=31, k_max=60)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    b = decode_batch(h, y, cfg, "fwbf", flip_log=True, force_ordered=NOFILTER)
    _same(a, b, f"tiny {tiny}")
    assert a.flip_logs() == b.flip_logs()
    _vs_oracle(a, h, y, cfg, f"tiny {tiny}")
