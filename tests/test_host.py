"""Host-side logic: config validation, code constructors, structure detection, I/O."""

import os

import numpy as np
import pytest

from paper_1206_3362_b200 import (DecoderConfig, ParityCheckMatrix, codes, detect_structure,
                                  eg_ldpc, gallager_rc, gf2_rank, pack_bits, qc_ldpc,
                                  read_alist, validate_rc, write_alist)
from paper_1206_3362_b200.sharding import frame_shard
from tests.golden.codebook import build_code, code_k
from tests.golden_io import GOLDEN


@pytest.mark.parametrize("kw,msg", [
    (dict(alpha=-0.1), "alpha"), (dict(k_max=0), "k_max"), (dict(lam=0), "lam"),
    (dict(block_len_p=0), "block_len_p"), (dict(stall_policy="x"), "stall_policy"),
    (dict(weight_mode="x"), "weight_mode")])
def test_decoder_config_errors_mirror_reference(kw, msg):
    # decoders.py:51-61
    with pytest.raises(ValueError, match=msg):
        DecoderConfig(**kw)


def test_eg_first_rows_and_ranks_match_reference():
    d = np.load(os.path.join(GOLDEN, "eg_first_rows.npz"))
    for s in (2, 3, 4, 5):
        h = eg_ldpc(s)
        assert np.array_equal(h.row_adj[0], d[f"s{s}"])
        assert gf2_rank(h) == int(d[f"rank{s}"])
        st = detect_structure(h)
        assert st.kind == "circulant" and np.array_equal(st.offsets, d[f"s{s}"])
        assert validate_rc(h)


def test_eg6_is_the_4095_3367_code():
    h = build_code("eg6")
    assert (h.n_rows, h.n_cols) == (4095, 4095)
    assert np.all(h.row_weights == 64) and np.all(h.col_weights == 64)
    assert h.n_cols - gf2_rank(h) == 3367 == code_k("eg6")


def test_qc_code_structure():
    h = build_code("qc4x32")
    st = detect_structure(h)
    assert st.kind == "qc" and st.z == 512 and st.shifts.shape == (4, 32)
    assert np.all(h.row_weights == 32) and np.all(h.col_weights == 4)
    assert validate_rc(h)                      # no 4-cycles
    assert h.n_cols - gf2_rank(h) == code_k("qc4x32")


def test_gallager_code():
    h = build_code("gal504")
    assert (h.n_rows, h.n_cols) == (252, 504)
    assert np.all(h.row_weights == 6) and np.all(h.col_weights == 3)
    assert validate_rc(h)
    assert detect_structure(h).kind == "explicit"


def test_matrix_views_consistent_and_syndrome():
    h = gallager_rc(60, 3, 6, seed=3)
    dense = h.to_dense()
    for n in range(h.n_cols):
        assert np.array_equal(h.col_adj[n], np.nonzero(dense[:, n])[0])
    rng = np.random.default_rng(0)
    z = rng.integers(0, 2, h.n_cols).astype(np.uint8)
    assert np.array_equal(h.syndrome(z), (dense.astype(int) @ z) % 2)
    with pytest.raises(ValueError):
        ParityCheckMatrix([[0, 0]], 3)
    with pytest.raises(ValueError):
        ParityCheckMatrix([[5]], 3)


def test_alist_round_trip(tmp_path):
    for h in (eg_ldpc(3), gallager_rc(60, 3, 6, seed=2)):
        p = tmp_path / "h.alist"
        write_alist(h, p)
        assert read_alist(p) == h
    bad = tmp_path / "bad.alist"
    bad.write_text("3 1\n1 3\n1 1 1\n2\n1\n1\n1\n1 2 3\n")
    with pytest.raises(codes.AlistError):
        read_alist(bad)


def test_pack_bits_layout():
    c = np.zeros(40, np.uint8)
    c[[0, 31, 32, 39]] = 1
    w = pack_bits(c, 40)
    assert w.tolist() == [1 | (1 << 31), 1 | (1 << 7)]


@pytest.mark.parametrize("count,world", [(10, 3), (0, 2), (1 << 20, 8), (7, 8)])
def test_frame_shards_tile_the_range(count, world):
    got = []
    for r in range(world):
        s, n = frame_shard(100, count, r, world)
        got.extend(range(s, s + n))
    assert got == list(range(100, 100 + count))
