"""Stage-level parity: the Eq.(1) metric vector the decode kernel computes in
its first iteration (fwbf_metric_*) equals the reference's all_metrics on the
initial state -- compute_weights + edge_weights + all_metrics,
decoders.py:80-103,148-153, restated in oracle/wbf_oracle.py -- bit for bit,
on every metric path (split-fp32, guarded fp64, ordered)."""

import numpy as np
import pytest

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.decoders import metric_batch
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import case_names, load_case

pytestmark = pytest.mark.gpu


def oracle_metric(h, y, alpha, weight_mode):
    g = O.Graph.of(h)
    out = np.empty((y.shape[0], g.n))
    for f in range(y.shape[0]):
        yf = np.asarray(y[f], dtype=np.float64)
        ay = np.abs(yf)
        synd = g.syndrome((yf < 0).astype(np.uint8))
        min1, min2, arg = O.check_minima(g, ay)
        ew = O.edge_weights(g, min1, min2, arg, weight_mode)
        out[f] = O.metric(g, synd, ew, ay, alpha)
    return out


def assert_bits_equal(a, b, tag):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    bad = np.nonzero(np.any(a.view(np.int64) != b.view(np.int64), axis=1))[0]
    assert bad.size == 0, f"{tag}: frames {bad[:8]} differ"


@pytest.mark.parametrize("ordered", [0, 1, 2], ids=["default", "ordered", "fp64guard"])
@pytest.mark.parametrize("name", case_names())
def test_metric_fixture(cuda_device, name, ordered):
    c = load_case(name)
    h = build_code(c.meta["code"])
    cfg = DecoderConfig(alpha=c.meta["alpha"], k_max=max(1, c.meta["k_max"]), lam=c.meta["lam"],
                        block_len_p=c.meta["p"], weight_mode=c.meta["weight_mode"])
    E, flags = metric_batch(h, c.y, cfg, c.meta["algorithm"], force_ordered=ordered)
    assert_bits_equal(E.cpu().numpy(), oracle_metric(h, c.y, cfg.alpha, cfg.weight_mode), name)
    fl = flags.cpu().numpy()
    if ordered == 1:
        assert np.all(fl & nat.FLAG_ORDERED)


@pytest.mark.parametrize("code,ebn0,dtype,weight_mode,alpha", [
    ("eg4", 2.0, np.float32, "imwbf", 0.2), ("eg5", 4.0, np.float32, "imwbf", 0.2),
    ("eg5", 3.0, np.float32, "mwbf", 0.0), ("eg5", 4.0, np.float64, "imwbf", 0.3),
    ("eg6", 4.0, np.float32, "imwbf", 0.2), ("gal504", 3.0, np.float32, "imwbf", 0.2),
    ("qc4x32", 5.0, np.float32, "imwbf", 0.2), ("qc4x32", 4.0, np.float64, "mwbf", 0.5)])
def test_metric_seeded(cuda_device, code, ebn0, dtype, weight_mode, alpha):
    h = build_code(code)
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    rng = np.random.default_rng(7)
    frames = 64 if h.n_cols <= 4096 else 8
    y = (1.0 + sigma * rng.standard_normal((frames, h.n_cols))).astype(dtype)
    cfg = DecoderConfig(alpha=alpha, k_max=5, block_len_p=32, weight_mode=weight_mode)
    for ordered in (0, 1):
        E, flags = metric_batch(h, y, cfg, "fwbf", force_ordered=ordered)
        assert_bits_equal(E.cpu().numpy(), oracle_metric(h, y, alpha, weight_mode), f"{code}/{ordered}")
    if dtype == np.float32 and code.startswith("eg"):
        # the default run took the split-fp32 path on (nearly) every frame
        E, flags = metric_batch(h, y, cfg, "fwbf")
        assert np.mean((flags.cpu().numpy() & nat.FLAG_SPLIT32) != 0) > 0.5


def test_metric_spec_weights_example(cuda_device):
    """N(m) = {1, 2, 3}, |y| = (0.5, 0.2, 0.9) -> w = (0.2, 0.5, 0.2),
    seen through the metric of a one-check code (E_n = +-w_n - alpha |y_n|)."""
    from paper_1206_3362_b200.codes import ParityCheckMatrix
    h = ParityCheckMatrix([[0, 1, 2]], 3)
    y = np.array([[0.5, -0.2, 0.9]], dtype=np.float32)       # one negative bit: s = 1
    E, _ = metric_batch(h, y, DecoderConfig(alpha=0.0, block_len_p=1))
    w = np.array([np.float32(0.2), np.float32(0.5), np.float32(0.2)], dtype=np.float64)
    assert np.array_equal(E.cpu().numpy()[0], w)


@pytest.mark.parametrize("code", ["eg5", "eg6"])
def test_metric_split_adversarial_lo_sum(cuda_device, code):
    """Every |y| = 2^e (1.0625 - 2^-23): on the split-fp32 grid each weight has
    a low part of G/2 - q, the largest possible.  With dv = 64 the low-part
    partial sums pass 2^24 q, so the grid must be G = 2^19 q there (2^20 q is
    exact only up to dv = 32).  The metric must still equal the reference's."""
    h = build_code(code)
    for e in (-10, 0, 3):
        v0 = np.float32(2.0 ** e * (1.0625 - 2.0 ** -23))
        y = np.full((2, h.n_cols), v0, dtype=np.float32)
        y[1, ::7] = -v0                                   # mixed syndromes too
        cfg = DecoderConfig(alpha=0.2, k_max=5, block_len_p=31)
        E, flags = metric_batch(h, y, cfg)
        assert_bits_equal(E.cpu().numpy(), oracle_metric(h, y, 0.2, "imwbf"), f"{code}/e={e}")
