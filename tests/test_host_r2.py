"""Host-side API pinned to reference-generated fixtures (tests/golden/make_golden_r2.py):
RC check reports, code_spec, alist error classes, the channel's per-frame API,
and write_csv byte identity."""

import json
import os

import numpy as np
import pytest

import paper_1206_3362_b200 as P
from paper_1206_3362_b200 import codes
from paper_1206_3362_b200.harness import PointStats, write_csv
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import GOLDEN


def _host_tools():
    with open(os.path.join(GOLDEN, "host_tools.json")) as f:
        return json.load(f)


def _pair(p):
    return None if p is None else tuple(p)


def test_validate_rc_reports_match_reference():
    d = _host_tools()
    for code, (ok, rp, cp) in d["rc"].items():
        h = codes.ParityCheckMatrix(d["bad_rows"], 6) if code == "bad" else build_code(code)
        r = P.validate_rc(h)
        assert isinstance(r, P.RcReport)
        assert (r.ok, r.row_pair, r.col_pair) == (ok, _pair(rp), _pair(cp)), code
        assert bool(r) == ok


def test_code_spec_matches_reference():
    d = _host_tools()
    for code, want in d["spec"].items():
        h = codes.ParityCheckMatrix(d["irregular_rows"], 5) if code == "irregular" else build_code(code)
        s = P.code_spec(h)
        assert [s.n, s.k, s.rate, s.row_weight, s.col_weight] == want, code
    assert P.code_spec(codes.ParityCheckMatrix([[0, 1], [0, 1]], 2)).k == 1
    with pytest.raises(ValueError, match="degenerate"):
        P.code_spec(codes.ParityCheckMatrix([[0], [1]], 2))          # k = 0


def test_alist_error_classes_match_reference(tmp_path):
    d = _host_tools()
    for name, case in d["alist"].items():
        p = tmp_path / f"{name}.alist"
        p.write_text(case["text"])
        if case["error"] is None:
            h = P.read_alist(p)
            assert [a.tolist() for a in h.row_adj] == case["rows"], name
        else:
            cls = getattr(P, case["error"])
            with pytest.raises(cls) as ei:
                P.read_alist(p)
            assert type(ei.value) is cls, (name, type(ei.value))
            assert isinstance(ei.value, P.AlistError) and isinstance(ei.value, ValueError)


def test_alist_roundtrip_and_transpose(tmp_path):
    h = build_code("gal504")
    P.write_alist(h, tmp_path / "g.alist")
    assert P.read_alist(tmp_path / "g.alist") == h
    t = h.transpose()
    assert (t.n_rows, t.n_cols) == (h.n_cols, h.n_rows)
    assert t.transpose() == h
    pad = h.row_pad
    assert pad.shape == (h.n_rows, h.max_row_weight) and np.all(pad[:, :6] == np.stack(h.row_adj))


def test_channel_host_api_matches_reference_stream():
    d = np.load(os.path.join(GOLDEN, "channel_normals.npz"))
    for key in d.files:
        seed, frame = map(int, key.split("_"))
        g = P.frame_rng(seed, frame).standard_normal(1023)
        assert np.array_equal(g, d[key]), key
    s = P.bpsk_modulate(np.array([0, 1, 1, 0], np.uint8))
    assert s.tolist() == [1.0, -1.0, -1.0, 1.0]
    with pytest.raises(ValueError):
        P.bpsk_modulate(np.array([0, 2]))
    with pytest.raises(ValueError):
        P.frame_rng(-1, 0)
    with pytest.raises(ValueError):
        P.awgn_apply(s, -0.1, P.frame_rng(1, 0))
    sigma = P.ebn0_to_sigma(4.0, code_rate("eg5"))
    fr = P.transmit(np.zeros(1023, np.uint8), sigma, P.frame_rng(1, 0))
    assert np.array_equal(fr.y, 1.0 + sigma * d["1_0"])
    assert np.array_equal(P.awgn_apply(s, 0.0, None), s)
    assert P.ChannelParams(4.0, 0.5).sigma == P.ebn0_to_sigma(4.0, 0.5)
    with pytest.raises(ValueError):
        P.ReceivedFrame(np.zeros(3), np.zeros(2))


def test_write_csv_byte_identical_to_reference(tmp_path):
    with open(os.path.join(GOLDEN, "experiment.json")) as f:
        meta = json.load(f)
    stats = [PointStats(**s) for s in meta["stats"]]
    write_csv(stats, tmp_path / "x.csv")
    with open(os.path.join(GOLDEN, "experiment.csv"), "rb") as f:
        want = f.read()
    assert (tmp_path / "x.csv").read_bytes() == want


def test_seed_range_checks():
    from paper_1206_3362_b200.harness import ExperimentConfig
    h = build_code("eg3")
    with pytest.raises(ValueError, match="master_seed"):
        ExperimentConfig(h=h, decoder="fwbf", decoder_cfg=P.DecoderConfig(block_len_p=8), ebn0_db=(3.0,),
                         master_seed=1 << 64)
