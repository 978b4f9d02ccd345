"""Property tests of the SPEC.md invariants on the CPU oracle (hypothesis), plus
the GPU versions of the same properties on small random codes (-m gpu)."""

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import eg_ldpc, gallager_rc

CODES = {"eg3": eg_ldpc(3), "eg4": eg_ldpc(4), "gal60": gallager_rc(60, 3, 6, seed=7)}


def frames(draw, n):
    sigma = draw(st.floats(0.3, 1.0))
    seed = draw(st.integers(0, 2 ** 31))
    rng = np.random.default_rng(seed)
    return (1.0 + sigma * rng.standard_normal(n)).astype(np.float32)


@settings(max_examples=60, deadline=None)
@given(st.data())
def test_fwbf_pN_equals_mlp_lambda1(data):
    # one block == lambda = 1 (same stall policy)
    name = data.draw(st.sampled_from(sorted(CODES)))
    g = O.Graph.of(CODES[name])
    y = frames(data.draw, g.n)
    stall = data.draw(st.sampled_from(["terminate", "flip-global-max"]))
    a = O.decode(g, y, "fwbf", p=g.n, k_max=15, stall=stall)
    b = O.decode(g, y, "mlp", lam=1, k_max=15, stall=stall)
    assert a.flip_log == b.flip_log and a.iterations == b.iterations


@settings(max_examples=60, deadline=None)
@given(st.data())
def test_positive_scaling_invariance(data):
    # exact power-of-two scaling keeps every decision
    name = data.draw(st.sampled_from(sorted(CODES)))
    g = O.Graph.of(CODES[name])
    y = frames(data.draw, g.n)
    c = data.draw(st.sampled_from([0.25, 0.5, 2.0, 8.0]))
    p = data.draw(st.integers(1, g.n))
    a = O.decode(g, y, "fwbf", p=p, k_max=15)
    b = O.decode(g, y * np.float32(c), "fwbf", p=p, k_max=15)
    assert a.flip_log == b.flip_log


@settings(max_examples=40, deadline=None)
@given(st.data())
def test_flip_count_bounds_and_syndrome_consistency(data):
    # incremental syndrome == recomputed; flips per iteration bounded
    name = data.draw(st.sampled_from(sorted(CODES)))
    g = O.Graph.of(CODES[name])
    y = frames(data.draw, g.n)
    p = data.draw(st.integers(1, g.n))
    r = O.decode(g, y, "fwbf", p=p, k_max=20)
    z = (y < 0).astype(np.uint8)
    for fl in r.flip_log:
        assert len(fl) <= -(-g.n // p)
        z[np.asarray(fl, dtype=np.int64)] ^= 1
    assert np.array_equal(z, r.z)
    assert r.converged == (not g.syndrome(r.z).any())
    assert r.iterations <= 20


def test_single_error_correction_exhaustive():
    # SPEC.md:271 / acceptance 6: every single hard error on EG(2,4) (n=15) is corrected
    h = eg_ldpc(2)
    g = O.Graph.of(h)
    for pos in range(g.n):
        y = np.ones(g.n)
        y[pos] = -0.8
        for alg, kw in (("imwbf", {}), ("fwbf", dict(p=4)), ("fwbf", dict(p=1))):
            r = O.decode(g, y, alg, k_max=10, **kw)
            assert r.converged and not r.z.any(), (pos, alg, kw)


# ---------------------------------------------------------------- GPU versions
def _batch(n, B, sigma, seed):
    rng = np.random.default_rng(seed)
    return (1.0 + sigma * rng.standard_normal((B, n))).astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("s", [5, 6])
def test_gpu_fwbf_pN_equals_mlp_lambda1(cuda_device, s):
    from paper_1206_3362_b200 import DecoderConfig, decode_batch
    h = eg_ldpc(s)
    y = _batch(h.n_cols, 512, 0.62, 11 + s)
    for stall in ("terminate", "flip-global-max"):
        a = decode_batch(h, y, DecoderConfig(alpha=0.2, k_max=30, block_len_p=h.n_cols,
                                              stall_policy=stall), "fwbf", flip_log=True)
        b = decode_batch(h, y, DecoderConfig(alpha=0.2, k_max=30, lam=1, stall_policy=stall),
                         "mlp", flip_log=True)
        assert a.flip_logs() == b.flip_logs()
        assert np.array_equal(a.iterations.cpu().numpy(), b.iterations.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("c", [0.5, 4.0])
def test_gpu_scaling_invariance(cuda_device, c):
    from paper_1206_3362_b200 import DecoderConfig, decode_batch
    h = eg_ldpc(5)
    y = _batch(h.n_cols, 2048, 0.6, 5)
    cfg = DecoderConfig(alpha=0.2, k_max=100, block_len_p=31)
    a = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    b = decode_batch(h, y * np.float32(c), cfg, "fwbf", flip_log=True)
    assert a.flip_logs() == b.flip_logs()


@pytest.mark.gpu
def test_gpu_syndrome_consistency_and_bounds(cuda_device):
    from paper_1206_3362_b200 import DecoderConfig, decode_batch
    h = eg_ldpc(5)
    g = O.Graph.of(h)
    y = _batch(h.n_cols, 256, 0.65, 9)
    p = 31
    res = decode_batch(h, y, DecoderConfig(alpha=0.2, k_max=100, block_len_p=p), "fwbf", flip_log=True)
    zs, logs, conv = res.z(), res.flip_logs(), res.converged
    for f in range(y.shape[0]):
        z = (y[f] < 0).astype(np.uint8)
        for fl in logs[f]:
            assert len(fl) <= -(-g.n // p)
            assert all((a // p) != (b // p) for a, b in zip(fl, fl[1:]))  # one flip per block
            z[np.asarray(fl, dtype=np.int64)] ^= 1
        assert np.array_equal(z, zs[f])
        assert conv[f] == (not g.syndrome(zs[f]).any())
