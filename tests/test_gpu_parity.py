"""CUDA path vs the reference (golden fixtures) and vs the CPU oracle.

Bit-exact: hard decisions, iteration counts, converged/stalled flags, flip
counts and the full flip sequence.  Both metric paths are checked: the
default (guarded fast path where the exactness guard holds) and
force_ordered (the reference's summation order everywhere).
"""

import numpy as np
import pytest

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import DecoderConfig, decode_batch, decode_fwbf, decode_imwbf, decode_mlp_wbf
from paper_1206_3362_b200 import _native as nat
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import case_names, load_case

pytestmark = pytest.mark.gpu


def cfg_of(meta):
    return DecoderConfig(alpha=meta["alpha"], k_max=meta["k_max"], lam=meta["lam"],
                         block_len_p=meta["p"], stall_policy=meta["stall"],
                         mlp_threshold=meta["mlp_threshold"], weight_mode=meta["weight_mode"])


def assert_batch_equal(res, z, iters, conv, stalled, flips_total, logs, tag):
    its = res.iterations.cpu().numpy()
    bad = np.nonzero((its != iters) | np.any(res.z() != z, axis=1) |
                     (res.converged != conv) | (res.stalled != stalled) |
                     (res.flips_total.cpu().numpy() != flips_total))[0]
    assert bad.size == 0, f"{tag}: frames {bad[:10]} differ"
    if logs is not None:
        got = res.flip_logs()
        for i, (a, b) in enumerate(zip(got, logs)):
            assert a == b, f"{tag}: flip log of frame {i} differs"


@pytest.mark.parametrize("ordered", [0, 1, 2, 4], ids=["default", "ordered", "fp64guard", "nofilter"])
@pytest.mark.parametrize("name", case_names())
def test_golden_fixture(cuda_device, name, ordered):
    c = load_case(name)
    h = build_code(c.meta["code"])
    res = decode_batch(h, c.y, cfg_of(c.meta), c.meta["algorithm"], flip_log=True,
                       force_ordered=ordered)
    assert_batch_equal(res, c.z, c.iterations, c.converged, c.stalled, c.flips_total,
                       c.flip_logs, name)


def _oracle_batch(h, y, alg, cfg):
    g = O.Graph.of(h)
    outs = [O.decode(g, y[i], alg, alpha=cfg.alpha, k_max=cfg.k_max, lam=cfg.lam,
                     p=cfg.block_len_p, stall=cfg.stall_policy, mlp_threshold=cfg.mlp_threshold,
                     weight_mode=cfg.weight_mode) for i in range(y.shape[0])]
    return (np.stack([o.z for o in outs]), np.array([o.iterations for o in outs]),
            np.array([o.converged for o in outs]), np.array([o.stalled for o in outs]),
            np.array([o.flips_total for o in outs]), [o.flip_log for o in outs])


def seeded_y(code, ebn0, frames, seed, dtype=np.float32):
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    rng = np.random.default_rng(seed)
    return h, (1.0 + sigma * rng.standard_normal((frames, h.n_cols))).astype(dtype)


@pytest.mark.parametrize("code,alg,kw,ebn0,frames", [
    ("eg5", "fwbf", dict(block_len_p=31, k_max=100), 4.0, 192),
    ("eg5", "fwbf", dict(block_len_p=93, k_max=100), 3.5, 96),
    ("eg5", "imwbf", dict(k_max=60), 4.0, 48),
    ("eg5", "mlp", dict(lam=10, k_max=100), 3.5, 64),
    ("eg4", "fwbf", dict(block_len_p=16, k_max=50, stall_policy="terminate"), 2.5, 512),
    ("eg4", "fwbf", dict(block_len_p=7, k_max=50, alpha=0.0, weight_mode="mwbf"), 3.0, 256),
    ("gal504", "fwbf", dict(block_len_p=24, k_max=50), 4.0, 256),
    ("gal504", "mlp", dict(lam=5, k_max=50, mlp_threshold=False), 4.0, 64),
])
def test_seeded_frames_vs_oracle(cuda_device, code, alg, kw, ebn0, frames):
    h, y = seeded_y(code, ebn0, frames, seed=hash((code, alg, ebn0)) & 0xffff)
    cfg = DecoderConfig(**kw)
    res = decode_batch(h, y, cfg, alg, flip_log=True)
    assert_batch_equal(res, *_oracle_batch(h, y, alg, cfg), f"{code}/{alg}")


def test_float64_input_vs_oracle(cuda_device):
    h, y = seeded_y("eg5", 4.0, 48, seed=11, dtype=np.float64)
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    res = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    assert_batch_equal(res, *_oracle_batch(h, y, "fwbf", cfg), "f64")
    assert np.all(res.flags.cpu().numpy() & nat.FLAG_ORDERED)


def test_per_frame_api_and_trace(cuda_device):
    c = load_case("B_fwbf_p31_40")
    h = build_code("eg5")
    cfg = cfg_of(c.meta)
    out = decode_fwbf(h, c.y[0], cfg, trace=True)
    assert out.iterations == c.iterations[0] and out.flip_log == c.flip_logs[0]
    assert len(out.trace) == out.iterations + 1
    for st in out.trace:                       # syndrome consistency
        assert np.array_equal(st.syndrome, h.syndrome(st.z))
    assert out.converged == (out.trace[-1].syndrome_weight == 0)
    o2 = decode_imwbf(h, c.y[1].astype(np.float64), DecoderConfig(k_max=5))
    r2 = O.decode(O.Graph.of(h), c.y[1], "imwbf", k_max=5)
    assert o2.flip_log == r2.flip_log
    o3 = decode_mlp_wbf(h, c.y[2], DecoderConfig(lam=3, k_max=5))
    r3 = O.decode(O.Graph.of(h), c.y[2], "mlp", lam=3, k_max=5)
    assert o3.flip_log == r3.flip_log and np.array_equal(o3.z_final, r3.z)
    with pytest.raises(ValueError):
        decode_mlp_wbf(h, c.y[0], DecoderConfig(lam=2000))
    with pytest.raises(ValueError):
        decode_fwbf(h, c.y[0], DecoderConfig())
    with pytest.raises(ValueError):
        decode_fwbf(h, c.y[0][:100], DecoderConfig(block_len_p=3))


# ---- full-size, size-independent properties (config B, 2^16 frames) ----------

@pytest.fixture(scope="module")
def big_b(cuda_device):
    import torch
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
    g = torch.Generator(device="cuda").manual_seed(1234)
    y = (1.0 + sigma * torch.randn((1 << 16, 1023), generator=g, device="cuda")).float()
    return h, y


def _summary(res):
    return (res.z_bits.cpu().numpy(), res.iterations.cpu().numpy(),
            res.flags.cpu().numpy() & 3, res.flips_total.cpu().numpy())


def test_guarded_equals_ordered_full_size(big_b):
    h, y = big_b
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    a = decode_batch(h, y, cfg, "fwbf")
    b = decode_batch(h, y, cfg, "fwbf", force_ordered=True)
    for u, v in zip(_summary(a), _summary(b)):
        assert np.array_equal(u, v)
    cnt = a.counters.cpu().numpy()
    assert cnt[nat.CNT_FRAMES] == y.shape[0]
    assert cnt[nat.CNT_ITER_SUM] == a.iterations.cpu().numpy().sum()
    assert cnt[nat.CNT_FLIP_SUM] == a.flips_total.cpu().numpy().sum()
    assert cnt[nat.CNT_BIT_ERRORS] == a.bit_errors.cpu().numpy().sum()
    assert cnt[nat.CNT_WORD_ERRORS] == (a.bit_errors.cpu().numpy() > 0).sum()
    # the guard is rare to fail: at most a few in 1e4 frames take the ordered path
    assert cnt[nat.CNT_ORDERED_FRAMES] < y.shape[0] * 1e-3


def test_split_fp32_equals_fp64_guarded_full_size(big_b):
    h, y = big_b
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    a = decode_batch(h, y, cfg, "fwbf")
    b = decode_batch(h, y, cfg, "fwbf", force_ordered=2)
    for u, v in zip(_summary(a), _summary(b)):
        assert np.array_equal(u, v)
    fl = a.flags.cpu().numpy()
    assert (fl & nat.FLAG_SPLIT32).mean() > 0.9      # most frames take the split-fp32 path
    assert not np.any(b.flags.cpu().numpy() & nat.FLAG_SPLIT32)


def test_scale_invariance_full_size(big_b):
    # positive scaling of y leaves every decision unchanged
    # (x2 is exact in float32, so every metric scales exactly).
    h, y = big_b
    cfg = DecoderConfig(block_len_p=93, k_max=100)
    a = decode_batch(h, y, cfg, "fwbf")
    b = decode_batch(h, y * 2.0, cfg, "fwbf")
    for u, v in zip(_summary(a), _summary(b)):
        assert np.array_equal(u, v)


def test_fwbf_pN_equals_mlp_lambda1(big_b):
    # FWBF with one block == MLP-WBF with lambda = 1
    h, y = big_b
    y = y[:8192]
    a = decode_batch(h, y, DecoderConfig(block_len_p=1023, k_max=30), "fwbf")
    b = decode_batch(h, y, DecoderConfig(lam=1, k_max=30), "mlp")
    for u, v in zip(_summary(a), _summary(b)):
        assert np.array_equal(u, v)


def test_converged_frames_satisfy_checks(big_b):
    h, y = big_b
    res = decode_batch(h, y[:4096], DecoderConfig(block_len_p=31, k_max=100), "fwbf")
    z = res.z()
    conv = res.converged
    syn = np.array([h.syndrome(z[i]).any() for i in range(z.shape[0])])
    assert np.array_equal(~syn, conv | (~syn & ~conv)) and not np.any(syn[conv])


def test_empty_batch(cuda_device):
    h = build_code("eg4")
    res = decode_batch(h, np.zeros((0, 255), np.float32), DecoderConfig(block_len_p=8), "fwbf")
    assert res.iterations.numel() == 0


def test_code_too_large_for_shared_memory_fails_cleanly(cuda_device):
    """Frame state lives in shared memory; a code beyond that fails with a
    clear error at decode time (no launch, no CPU fallback)."""
    from paper_1206_3362_b200.codes import ParityCheckMatrix
    n = 60000
    rows = [[(3 * r + k) % n for k in (0, 1, 2, 3, 4, 5)] for r in range(n // 2)]
    h = ParityCheckMatrix([sorted(set(r)) for r in rows], n)
    y = np.ones((2, n), np.float32)
    with pytest.raises((nat.FwbfError, ValueError), match="shared memory|fit"):
        decode_batch(h, y, DecoderConfig(block_len_p=24, k_max=3), "fwbf")


def test_single_frame_extremes(cuda_device):
    """One frame each: all +1 (converged at k = 0), all -1, all exact zeros and
    alternating signs, on the split, guarded and ordered paths; vs the oracle."""
    h = build_code("eg5")
    n = h.n_cols
    ys = np.stack([np.ones(n), -np.ones(n), np.zeros(n), np.where(np.arange(n) % 2, 1.0, -1.0),
                   np.full(n, 1e-30), np.linspace(-3, 3, n), np.linspace(-3e35, 2e35, n),
                   np.where(np.arange(n) % 3, 1e34, -2e33), np.full(n, -1e-40),
                   np.where(np.arange(n) % 5, 3e-41, -1e30), np.where(np.arange(n) % 2, 1.0, -0.0)
                   ]).astype(np.float32)
    cfg = DecoderConfig(block_len_p=31, k_max=30)
    exp = _oracle_batch(h, ys, "fwbf", cfg)
    for ordered in (0, 1, 2):
        res = decode_batch(h, ys, cfg, "fwbf", flip_log=True, force_ordered=ordered)
        assert_batch_equal(res, *exp, f"extremes/{ordered}")
