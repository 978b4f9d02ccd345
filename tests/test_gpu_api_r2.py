"""Device-backed stage API, channel batch, harness workflow and host-interface
fixes, checked against reference-generated fixtures (make_golden_r2.py) and
the pinned oracle."""

import json
import os

import numpy as np
import pytest

import paper_1206_3362_b200 as P
from oracle import wbf_oracle as O
from paper_1206_3362_b200 import harness as H
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import GOLDEN

pytestmark = pytest.mark.gpu


def _sv():
    return np.load(os.path.join(GOLDEN, "stage_vectors.npz"))


@pytest.mark.parametrize("code", ["eg4", "gal504", "eg3"])
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_stage_functions_match_reference(cuda_device, code, tag):
    d = _sv()
    k = f"{code}_{tag}"
    h = build_code(code)
    Y = d[f"{k}_y"]
    for i in range(Y.shape[0]):
        z = P.hard_decision(Y[i])
        assert z.dtype == np.uint8 and np.array_equal(z, d[f"{k}_z"][i])
        assert np.array_equal(P.syndrome(h, z), d[f"{k}_syn"][i])
        w = P.compute_weights(h, Y[i])
        assert np.array_equal(w.min1, d[f"{k}_min1"][i])
        assert np.array_equal(w.min2, d[f"{k}_min2"][i])
        assert np.array_equal(w.argmin_col, d[f"{k}_argmin"][i])
        ew = w.edge_weights(h)
        assert np.array_equal(ew, d[f"{k}_edge_w"][i])
        ay = np.abs(Y[i].astype(np.float64))
        m = P.all_metrics(h, d[f"{k}_syn"][i], ew, ay, 0.2)
        assert np.array_equal(m, d[f"{k}_metric"][i])                 # bit-exact fp64
        m2 = P.all_metrics(h, d[f"{k}_syn2"][i], ew, ay, 0.7)
        assert np.array_equal(m2, d[f"{k}_metric2"][i])
        st = P.DecodeState(d[f"{k}_z2"][i], d[f"{k}_syn2"][i], 0)
        for j, c in enumerate(d[f"{k}_bm_cols"]):
            assert P.bit_metric(h, int(c), st, w, Y[i], 0.7) == d[f"{k}_bit_metric"][i, j]
    # batched forms: one launch over all frames, same values
    wb = P.compute_weights(h, Y)
    assert np.array_equal(wb.min1, d[f"{k}_min1"]) and np.array_equal(wb.argmin_col, d[f"{k}_argmin"])
    assert np.array_equal(wb.edge_weights(h), d[f"{k}_edge_w"])
    mb = P.all_metrics(h, d[f"{k}_syn"], d[f"{k}_edge_w"], np.abs(Y.astype(np.float64)), 0.2)
    assert np.array_equal(mb, d[f"{k}_metric"])
    assert np.array_equal(P.syndrome(h, d[f"{k}_z"]), d[f"{k}_syn"])


def test_block_argmax_matches_reference(cuda_device):
    d = _sv()
    for vk in ("ties", "neg", "nan", "rand"):
        v = d[f"ba_{vk}_v"]
        for p in (1, 2, 3, 7, 16, 255, 1000):
            got = P.block_argmax(v, p)
            assert got.dtype == np.int64 and np.array_equal(got, d[f"ba_{vk}_p{p}"]), (vk, p)
    with pytest.raises(ValueError):
        P.block_argmax(np.zeros(4), 0)


def test_stage_errors_mirror_reference(cuda_device):
    h = P.ParityCheckMatrix([[0, 1], [2]], 3)    # a check with one bit
    with pytest.raises(ValueError, match="at least 2 bits"):
        P.compute_weights(h, np.ones(3))
    with pytest.raises(ValueError, match="length"):
        P.compute_weights(build_code("eg3"), np.ones(5))


def test_stage_tensors_stay_on_device(cuda_device):
    import torch
    h = build_code("eg4")
    y = torch.randn(64, h.n_cols, device="cuda", dtype=torch.float64)
    z = P.hard_decision(y)
    assert isinstance(z, torch.Tensor) and z.is_cuda
    w = P.compute_weights(h, y)
    assert w.min1.is_cuda and w.min1.shape == (64, h.n_rows)
    e = P.block_argmax(y, 16)
    assert e.is_cuda and e.shape == (64, 16)


def test_awgn_batch_equals_reference_stream(cuda_device):
    d = np.load(os.path.join(GOLDEN, "channel_normals.npz"))
    h = build_code("eg5")
    sigma = P.ebn0_to_sigma(4.0, code_rate("eg5"))
    y = P.awgn_batch(h, 1, 0, 2, sigma).cpu().numpy()
    for f in range(2):
        want = 1.0 + sigma * d[f"1_{f}"]
        # <= 2 ulp on tail samples (CUDA log1p vs glibc), see test_gpu_noise.py
        assert np.all(np.abs(y[f] - want) <= 2 * np.spacing(np.abs(want)))
        assert np.mean(y[f] == want) > 0.999
    y32 = P.awgn_batch(h, 1, 0, 2, sigma, noise="f32").cpu().numpy()
    assert y32.dtype == np.float32 and np.array_equal(y32, y.astype(np.float32))
    cw = np.zeros(h.n_cols, np.uint8)
    cw[::3] = 1
    yc = P.awgn_batch(h, 1, 0, 2, 0.0, codeword=cw).cpu().numpy()
    assert np.array_equal(yc[0], 1.0 - 2.0 * cw)
    with pytest.raises(ValueError):
        P.awgn_batch(h, 1 << 64, 0, 2, sigma)


def test_run_experiment_csv_byte_identical_to_reference(cuda_device, tmp_path):
    with open(os.path.join(GOLDEN, "experiment.json")) as f:
        m = json.load(f)
    h = build_code(m["code"])
    path = tmp_path / "gpu.csv"
    ec = H.ExperimentConfig(h=h, decoder=m["decoder"], decoder_cfg=P.DecoderConfig(**m["cfg"]),
                            ebn0_db=tuple(m["ebn0_db"]), target_word_errors=m["target_word_errors"],
                            max_frames=m["max_frames"], master_seed=m["master_seed"], out_path=str(path),
                            chunk_frames=384)
    stats = H.run_experiment(ec)
    assert [s.__dict__ for s in stats] == m["stats"]
    with open(os.path.join(GOLDEN, "experiment.csv"), "rb") as f:
        assert path.read_bytes() == f.read()


def test_sweep_alpha_and_mlp_point_match_reference(cuda_device):
    with open(os.path.join(GOLDEN, "sweep_alpha.json")) as f:
        m = json.load(f)
    h = build_code(m["code"])
    ec = H.ExperimentConfig(h=h, decoder=m["decoder"], decoder_cfg=P.DecoderConfig(**m["cfg"]),
                            ebn0_db=(m["snr"],), target_word_errors=m["target_word_errors"],
                            max_frames=m["max_frames"], master_seed=m["master_seed"])
    sw = H.sweep_alpha(ec, m["grid"])
    assert sw.best_alpha == m["best_alpha"]
    assert [[a, s.__dict__] for a, s in sw.entries] == m["entries"]
    mp = m["mlp_point"]
    ec2 = H.ExperimentConfig(h=h, decoder="mlp", decoder_cfg=P.DecoderConfig(**mp["cfg"]), ebn0_db=(mp["snr"],),
                             target_word_errors=mp["target_word_errors"], max_frames=mp["max_frames"],
                             master_seed=mp["master_seed"], codeword=np.zeros(h.n_cols, np.uint8))
    assert H.run_point(ec2, mp["snr"]).__dict__ == mp["stats"]


def test_iteration_histogram(cuda_device):
    """Config E's iteration histogram: iter_hist[k] = frames that stopped after
    k iterations; equals the histogram of the per-frame counts (and the
    oracle's on a sample)."""
    import torch
    h = build_code("eg5")
    sigma = P.ebn0_to_sigma(4.0, code_rate("eg5"))
    cfg = P.DecoderConfig(block_len_p=31, k_max=100)
    res = P.decode_awgn(h, cfg, "fwbf", 1, 0, 1 << 14, sigma, noise="f32")
    hist = res.iter_hist.cpu().numpy()
    its = res.iterations.cpu().numpy()
    assert hist.shape == (101,) and hist.sum() == its.size
    assert np.array_equal(hist, np.bincount(its, minlength=101))
    assert int((hist * np.arange(101)).sum()) == int(res.counters[P.decoders.nat.CNT_ITER_SUM])
    y = P.awgn_batch(h, 1, 0, 64, sigma, noise="f32").cpu().numpy()
    g = O.Graph.of(h)
    ref = [O.decode(g, y[i], "fwbf", alpha=0.2, k_max=100, p=31).iterations for i in range(64)]
    assert np.array_equal(its[:64], ref)
    b = P.decode_batch(h, torch.from_numpy(y).cuda(), cfg)
    assert np.array_equal(b.iter_hist.cpu().numpy(), np.bincount(ref, minlength=101))


def test_redundant_h_more_checks_than_32_rounds(cuda_device):
    """M > 32 T used to overflow the per-thread syndrome register.
    A redundant H (every check duplicated many times, M >> 4N) must decode
    exactly like the oracle."""
    rng = np.random.default_rng(5)
    base = build_code("eg3")                       # 63 x 63
    rows = [r for r in base.row_adj] * 40           # M = 2520 > 32 * 64
    h = P.ParityCheckMatrix(rows, base.n_cols)
    sigma = O.ebn0_to_sigma(2.5, 37 / 63)
    y = (1.0 + sigma * rng.standard_normal((48, 63))).astype(np.float32)
    for alg, kw in (("fwbf", dict(block_len_p=8)), ("imwbf", {}), ("mlp", dict(lam=3))):
        cfg = P.DecoderConfig(k_max=20, **kw)
        res = P.decode_batch(h, y, cfg, alg, flip_log=True)
        logs = res.flip_logs()
        g = O.Graph.of(h)
        for i in range(y.shape[0]):
            r = O.decode(g, y[i], alg, alpha=0.2, k_max=20, p=kw.get("block_len_p"), lam=kw.get("lam", 1))
            assert int(res.iterations[i]) == r.iterations and logs[i] == r.flip_log, (alg, i)


def test_calls_restore_current_device(cuda_device):
    import torch
    torch.cuda.set_device(0)
    h = build_code("eg4")
    P.decode_batch(h, np.ones((2, 255), np.float32), P.DecoderConfig(block_len_p=16), device="cuda:0")
    assert torch.cuda.current_device() == 0
    P.device_code(h, 0).filter_stats()
    assert torch.cuda.current_device() == 0


def test_decode_on_side_stream_orders_inputs(cuda_device):
    """decode_batch(stream=s) waits for the inputs copied on the current stream."""
    import torch
    h = build_code("eg5")
    sigma = P.ebn0_to_sigma(4.0, code_rate("eg5"))
    y = P.awgn_batch(h, 3, 0, 4096, sigma, noise="f32")
    cfg = P.DecoderConfig(block_len_p=31, k_max=100)
    ref = P.decode_batch(h, y, cfg)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    yh = y.cpu().pin_memory()
    res = P.decode_batch(h, yh, cfg, stream=s)    # H2D copy on the current stream
    s.synchronize()
    assert torch.equal(res.iterations, ref.iterations) and torch.equal(res.z_bits, ref.z_bits)


@pytest.mark.parametrize("code,alg,kw", [
    ("eg4", "fwbf", dict(block_len_p=16, k_max=30)), ("eg5", "fwbf", dict(block_len_p=31, k_max=100)),
    ("eg5", "fwbf", dict(block_len_p=93, k_max=100, stall_policy="terminate")),
    ("eg5", "imwbf", dict(k_max=60)), ("eg5", "mlp", dict(lam=10, k_max=60)),
    ("eg5", "imwbf", dict(k_max=60, weight_mode="mwbf", alpha=0.0)), ("eg6", "fwbf", dict(block_len_p=64, k_max=60))])
@pytest.mark.parametrize("frames", [1, 37, 5000])
def test_staged_rows_equal_unstaged(cuda_device, monkeypatch, code, alg, kw, frames):
    """Rows with a 16-byte-multiple stride are staged into shared memory by a
    TMA bulk copy one frame ahead (row 27 of the scope table); the results
    must equal the element-wise load path, frame by frame and in the flip log."""
    import torch
    h = build_code(code)
    n = h.n_cols
    ld = (n + 3) // 4 * 4
    sigma = O.ebn0_to_sigma(3.5, code_rate(code))
    g = torch.Generator(device="cuda").manual_seed(frames)
    buf = torch.full((frames, ld), float("nan"), dtype=torch.float32, device="cuda")  # pad never read as data
    y = buf[:, :n]
    y.copy_(1.0 + sigma * torch.randn((frames, n), generator=g, device="cuda"))
    cfg = P.DecoderConfig(**kw)
    monkeypatch.setenv("FWBF_FORCE_YSTAGE", "1")   # staging also for the small batches
    a = P.decode_batch(h, y, cfg, alg, flip_log=True)
    monkeypatch.setenv("FWBF_NO_YSTAGE", "1")
    b = P.decode_batch(h, y, cfg, alg, flip_log=True)
    for name in ("z_bits", "iterations", "flags", "flips_total", "counters", "iter_hist"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert a.flip_logs() == b.flip_logs()
