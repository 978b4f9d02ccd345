"""Pin the CPU oracle to the reference: every golden fixture, bit for bit."""

import json
import os

import numpy as np
import pytest

from oracle import wbf_oracle as O
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import GOLDEN, case_names, load_case

# C/D fixtures take a few seconds each in numpy; still well within budget.
CASES = case_names()


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_fixture(name):
    c = load_case(name)
    g = O.Graph.of(build_code(c.meta["code"]))
    for i in range(c.y.shape[0]):
        r = O.decode(g, c.y[i], c.meta["algorithm"], **c.decoder_kwargs)
        assert np.array_equal(r.z, c.z[i]), (name, i)
        assert r.iterations == c.iterations[i], (name, i)
        assert r.converged == c.converged[i]
        assert r.stalled == c.stalled[i]
        assert r.flip_log == c.flip_logs[i], (name, i)
        assert r.flips_total == c.flips_total[i]


def test_oracle_channel_normals_match_reference():
    d = np.load(os.path.join(GOLDEN, "channel_normals.npz"))
    for key in d.files:
        seed, frame = map(int, key.split("_"))
        assert np.array_equal(O.frame_noise(seed, frame, 1023), d[key])


def test_oracle_run_batch_matches_reference():
    with open(os.path.join(GOLDEN, "run_batch.json")) as f:
        runs = json.load(f)
    g = O.Graph.of(build_code("eg5"))
    for r in runs[:1]:
        cfg = dict(k_max=r["cfg"]["k_max"], p=r["cfg"].get("block_len_p"), lam=r["cfg"].get("lam", 1))
        got = O.run_batch(g, r["algorithm"], r["sigma"], r["seed"], r["start"], r["count"], **cfg)
        assert list(got) == r["result"]


def test_sigma_known_answers():
    # SPEC.md:146-148 and BASELINE.md's config-B table
    assert O.ebn0_to_sigma(0.0, 0.5) == 1.0
    for db, s in [(3.0, 0.57292), (3.5, 0.54088), (4.0, 0.51062), (4.5, 0.48206), (5.0, 0.45509)]:
        assert abs(O.ebn0_to_sigma(db, code_rate("eg5")) - s) < 1e-5


def test_weights_spec_example():
    # N(m)={1,2,3}, |y|=(0.5,0.2,0.9) -> w = (0.2, 0.5, 0.2)
    g = O.Graph([[0, 1, 2]], 3)
    m1, m2, a = O.check_minima(g, np.array([0.5, 0.2, 0.9]))
    w = O.edge_weights(g, m1, m2, a)
    assert w.tolist() == [0.2, 0.5, 0.2]


@pytest.mark.parametrize("name", CASES)
def test_c_oracle_matches_reference_fixture(name):
    from oracle.c_oracle import COracle
    c = load_case(name)
    co = COracle(build_code(c.meta["code"]))
    z, its, fl, ft = co.decode_batch(c.y, algorithm=c.meta["algorithm"], **c.decoder_kwargs)
    assert np.array_equal(z, c.z), name
    assert np.array_equal(its, c.iterations), name
    assert np.array_equal((fl & 1).astype(bool), c.converged)
    assert np.array_equal((fl & 2).astype(bool), c.stalled)
    assert np.array_equal(ft, c.flips_total)
