"""Randomised parity: random small codes (regular, irregular, circulant), random
decoder knobs, random inputs (including ties and zeros) -- CUDA vs oracle, bit-exact."""

import os

import numpy as np
import pytest

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import DecoderConfig, ParityCheckMatrix, decode_batch, eg_ldpc, gallager_rc

pytestmark = pytest.mark.gpu


def random_code(rng):
    kind = rng.integers(0, 6)
    if kind == 4:  # the compile-time-weight kernels of the configs
        return eg_ldpc(int(rng.choice([4, 5])))
    if kind == 5:  # random circulant with a compiled-in weight (16 or 32) and an arbitrary n
        w = int(rng.choice([16, 32, 64]))
        n = int(rng.integers(w + 8, {16: 256, 32: 1024, 64: 4096}[w]))
        first = np.sort(rng.choice(n, size=w, replace=False))
        return ParityCheckMatrix([(first + i) % n for i in range(n)], n)
    if kind == 0:
        return eg_ldpc(int(rng.integers(2, 5)))
    if kind == 1:
        dv = int(rng.choice([2, 3, 4]))
        dc = int(rng.choice([4, 6, 8]))
        n = dc * int(rng.integers(4, 20))
        try:
            return gallager_rc(n, dv, dc, seed=int(rng.integers(1 << 30)))
        except RuntimeError:
            return eg_ldpc(3)
    if kind == 2:  # irregular random rows (weights 2..7), possibly with 4-cycles
        n = int(rng.integers(10, 120))
        m = int(rng.integers(3, n))
        rows = [np.sort(rng.choice(n, size=int(rng.integers(2, min(8, n) + 1)), replace=False))
                for _ in range(m)]
        return ParityCheckMatrix(rows, n)
    # circulant from a random offset set (not necessarily RC-free)
    n = int(rng.integers(20, 300))
    w = int(rng.integers(2, 12))
    first = np.sort(rng.choice(n, size=w, replace=False))
    return ParityCheckMatrix([(first + i) % n for i in range(n)], n)


def random_y(rng, n, frames):
    sigma = float(rng.uniform(0.3, 0.9))
    y = 1.0 + sigma * rng.standard_normal((frames, n))
    mode = rng.integers(0, 5)
    if mode == 1:
        y = np.round(y * 4) / 4  # ties and exact zeros
    elif mode == 3:  # per-frame power-of-two scale, far from 1 (guard and split boundaries)
        y = y * (2.0 ** rng.integers(-90, 91, size=(frames, 1)))
    elif mode == 4:  # heavy tails: a wide spread of exponents inside one frame
        y = y / np.maximum(rng.random((frames, n)), 1e-6) ** 2
    y = y.astype(np.float32 if rng.integers(0, 2) else np.float64)
    return y


@pytest.mark.parametrize("seed", range(int(os.environ.get("FWBF_FUZZ_N", "120"))))
def test_random_parity(cuda_device, seed):
    rng = np.random.default_rng(1000 + seed)
    h = random_code(rng)
    n = h.n_cols
    alg = ["fwbf", "imwbf", "mlp"][int(rng.integers(0, 3))]
    cfg = DecoderConfig(alpha=float(rng.choice([0.0, 0.2, 0.7, 1.5])), k_max=int(rng.integers(1, 40)),
                        lam=int(rng.integers(1, min(12, n) + 1)), block_len_p=int(rng.integers(1, n + 8)),
                        stall_policy=["flip-global-max", "terminate"][int(rng.integers(0, 2))],
                        mlp_threshold=bool(rng.integers(0, 2)),
                        weight_mode=["imwbf", "mwbf"][int(rng.integers(0, 2))])
    y = random_y(rng, n, int(rng.integers(1, 40)))
    res = decode_batch(h, y, cfg, alg, flip_log=True)
    z = res.z()
    its = res.iterations.cpu().numpy()
    logs = res.flip_logs()
    g = O.Graph.of(h)
    for i in range(y.shape[0]):
        r = O.decode(g, y[i], alg, alpha=cfg.alpha, k_max=cfg.k_max, lam=cfg.lam, p=cfg.block_len_p,
                     stall=cfg.stall_policy, mlp_threshold=cfg.mlp_threshold, weight_mode=cfg.weight_mode)
        assert its[i] == r.iterations, (seed, i)
        assert logs[i] == r.flip_log, (seed, i)
        assert np.array_equal(z[i], r.z), (seed, i)
        assert res.converged[i] == r.converged and res.stalled[i] == r.stalled


@pytest.mark.parametrize("seed", range(int(os.environ.get("FWBF_FUZZ_QC_N", "48"))))
def test_random_qc_parity(cuda_device, seed):
    """Random quasi-cyclic codes (2-4 row blocks, 3-40 block columns, absent
    blocks, Z = 32 / 64 / 128) with a block length the QC kernels accept
    (32 | p, p | Z): the incremental QC kernel (float32 input) or the generic
    path (float64 input) against the oracle, bit-exact, flip sequence included."""
    from paper_1206_3362_b200.codes import qc_from_shifts
    rng = np.random.default_rng(77000 + seed)
    jb, kb = int(rng.integers(2, 5)), int(rng.integers(3, 41))
    z = int(rng.choice([32, 64, 128]))
    sh = rng.integers(0, z, size=(jb, kb))
    if rng.integers(0, 2):
        full = sh.copy()
        sh[rng.random((jb, kb)) < 0.25] = -1
        sh[0, :] = full[0, :]                         # every column keeps a check
        for r in range(jb):                           # every check keeps at least two bits
            if np.count_nonzero(sh[r] >= 0) < 2:
                sh[r, :2] = full[r, :2]
    h = qc_from_shifts(sh, z)
    p = int(rng.choice([q for q in (32, 64, 128) if z % q == 0]))
    cfg = DecoderConfig(alpha=float(rng.choice([0.0, 0.2, 0.7, 1.5])), k_max=int(rng.integers(1, 30)),
                        block_len_p=p, stall_policy=["flip-global-max", "terminate"][int(rng.integers(0, 2))],
                        weight_mode=["imwbf", "mwbf"][int(rng.integers(0, 2))])
    y = random_y(rng, h.n_cols, int(rng.integers(1, 10)))
    res = decode_batch(h, y, cfg, "fwbf", flip_log=True)
    z_, its, logs = res.z(), res.iterations.cpu().numpy(), res.flip_logs()
    g = O.Graph.of(h)
    for i in range(y.shape[0]):
        r = O.decode(g, y[i], "fwbf", alpha=cfg.alpha, k_max=cfg.k_max, p=p, stall=cfg.stall_policy,
                     weight_mode=cfg.weight_mode)
        assert its[i] == r.iterations, (seed, i)
        assert logs[i] == r.flip_log, (seed, i)
        assert np.array_equal(z_[i], r.z), (seed, i)
        assert res.converged[i] == r.converged and res.stalled[i] == r.stalled
