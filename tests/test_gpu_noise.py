"""On-device reference channel (numpy Philox + ziggurat) and the GPU harness.

The device must reproduce channel.py's float64 y for every frame; the GPU
_run_batch / run_point must reproduce the reference harness' tuples and
statistics (golden run_batch.json from the reference, and the CPU oracle).
"""

import json
import os

import numpy as np
import pytest

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import harness as H
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate
from tests.golden_io import GOLDEN

pytestmark = pytest.mark.gpu


def _ulps(a, b):
    return np.abs(a.view(np.int64) - b.view(np.int64))


@pytest.mark.parametrize("seed,first,frames", [(1, 0, 3000), (7, 1 << 40, 300), (123456789, 12345, 300)])
def test_device_channel_matches_numpy(cuda_device, seed, first, frames):
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
    res = decode_awgn(h, DecoderConfig(block_len_p=31, k_max=1), "fwbf", seed, first, frames, sigma,
                      return_y=True)
    y = res.y.cpu().numpy()
    ref = np.stack([O.channel_frame(np.zeros(1023, np.uint8), sigma, seed, first + i)
                    for i in range(frames)])
    diff = y != ref
    # CUDA's log1p may round the tail sample (|g| > 3.65) one ulp away from glibc's
    assert diff.sum() <= max(2, frames * 1023 * 2e-5), diff.sum()
    if diff.any():
        assert np.all(_ulps(y[diff], ref[diff]) <= 2)
        assert np.all(np.abs(ref[diff] - 1.0) > 3.6 * sigma)


def test_device_channel_float32_and_codeword(cuda_device):
    h = build_code("eg4")
    sigma = O.ebn0_to_sigma(3.0, code_rate("eg4"))
    from paper_1206_3362_b200.codes import gf2_rank
    cw = np.zeros(255, np.uint8)  # all-zero is always a codeword; also a nonzero one:
    g = h.to_dense()
    # a nonzero codeword from the null space: use the all-ones word if it satisfies H
    ones = np.ones(255, np.uint8)
    if not h.syndrome(ones).any():
        cw = ones
    res = decode_awgn(h, DecoderConfig(block_len_p=16, k_max=30), "fwbf", 5, 0, 64, sigma,
                      codeword=cw, noise="f32", return_y=True)
    y = res.y.cpu().numpy()
    ref = np.stack([O.channel_frame(cw, sigma, 5, i) for i in range(64)]).astype(np.float32)
    assert (y != ref).sum() <= 2
    # decoding the generated values must equal decoding them from HBM
    b = decode_batch(h, y, DecoderConfig(block_len_p=16, k_max=30), "fwbf", codeword=cw)
    assert np.array_equal(b.iterations.cpu().numpy(), res.iterations.cpu().numpy())
    assert np.array_equal(b.bit_errors.cpu().numpy(), res.bit_errors.cpu().numpy())


def test_run_batch_matches_reference_tuples(cuda_device):
    with open(os.path.join(GOLDEN, "run_batch.json")) as f:
        runs = json.load(f)
    h = build_code("eg5")
    for r in runs:
        cfg = DecoderConfig(**r["cfg"])
        got = H._run_batch(h, r["algorithm"], cfg, r["sigma"], r["seed"], r["start"], r["count"], None)
        assert list(got) == r["result"], r


def test_run_batch_matches_oracle_larger(cuda_device):
    h = build_code("eg4")
    sigma = O.ebn0_to_sigma(2.5, code_rate("eg4"))
    cfg = DecoderConfig(block_len_p=16, k_max=40)
    got = H._run_batch(h, "fwbf", cfg, sigma, 3, 256, 512, None)
    ref = O.run_batch(O.Graph.of(h), "fwbf", sigma, 3, 256, 512, p=16, k_max=40)
    assert tuple(got) == tuple(ref)


def test_run_point_stop_rule_matches_oracle(cuda_device, tmp_path):
    h = build_code("eg4")
    cfg = DecoderConfig(block_len_p=16, k_max=30)
    conf = H.ExperimentConfig(h=h, decoder="fwbf", decoder_cfg=cfg, ebn0_db=(3.0,), rate=175 / 255,
                              target_word_errors=25, max_frames=5000, master_seed=2,
                              chunk_frames=384)
    st = H.run_point(conf, 3.0)
    # reference semantics: whole 128-frame batches until cumulative word errors >= 25
    sigma = O.ebn0_to_sigma(3.0, 175 / 255)
    g = O.Graph.of(h)
    tot = np.zeros(6, np.int64)
    for s in range(0, 5000, 128):
        tot += np.array(O.run_batch(g, "fwbf", sigma, 2, s, min(128, 5000 - s), p=16, k_max=30))
        if tot[2] >= 25:
            break
    assert (st.frames, st.bit_errors, st.word_errors, st.stalls) == (tot[0], tot[1], tot[2], tot[5])
    assert st.mean_iters == tot[3] / tot[0] and st.mean_flips == tot[4] / tot[0]
    assert not st.capped
    H.write_csv([st], tmp_path / "r.csv")
    assert (tmp_path / "r.csv").read_text().splitlines()[0] == H.CSV_HEADER


def test_sigma_zero_noiseless(cuda_device):
    h = build_code("eg4")
    res = decode_awgn(h, DecoderConfig(block_len_p=16), "fwbf", 1, 0, 256, 0.0, return_y=True)
    assert np.all(res.y.cpu().numpy() == 1.0)
    assert np.all(res.iterations.cpu().numpy() == 0)


def test_decode_awgn_concurrent_streams_share_scratch(cuda_device):
    """Two decode_awgn calls on different streams share the handle's y scratch;
    the library orders them on the device, so both results equal serial runs."""
    import torch
    from paper_1206_3362_b200 import DecoderConfig, eg_ldpc
    from paper_1206_3362_b200.decoders import decode_awgn
    h = eg_ldpc(5)
    cfg = DecoderConfig(block_len_p=31, k_max=50)
    ref_a = decode_awgn(h, cfg, "fwbf", 7, 0, 20000, 0.52)
    ref_b = decode_awgn(h, cfg, "fwbf", 9, 0, 20000, 0.55)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(sa):
        ra = decode_awgn(h, cfg, "fwbf", 7, 0, 20000, 0.52)
    with torch.cuda.stream(sb):
        rb = decode_awgn(h, cfg, "fwbf", 9, 0, 20000, 0.55)
    torch.cuda.synchronize()
    assert torch.equal(ra.iterations, ref_a.iterations) and torch.equal(ra.z_bits, ref_a.z_bits)
    assert torch.equal(rb.iterations, ref_b.iterations) and torch.equal(rb.z_bits, ref_b.z_bits)


def test_decode_awgn_two_stream_chunks_equal_single_chunks(cuda_device):
    """Batches larger than one chunk rotate three scratch buffers over two
    streams (deferred-frame launches on a third); with six chunks every buffer
    is reused.  Every frame's result and the accumulated counters equal those
    of single-chunk calls over the same frame ranges."""
    import torch
    from paper_1206_3362_b200 import DecoderConfig
    from paper_1206_3362_b200.decoders import decode_awgn
    from tests.golden.codebook import build_code, code_rate
    h = build_code("eg5")
    sigma = O.ebn0_to_sigma(4.5, code_rate("eg5"))
    cfg = DecoderConfig(block_len_p=31, k_max=60)
    whole = decode_awgn(h, cfg, "fwbf", 7, 1000, 700000, sigma, noise="f32")
    parts = [decode_awgn(h, cfg, "fwbf", 7, 1000 + s, 100000, sigma, noise="f32") for s in range(0, 700000, 100000)]
    torch.cuda.synchronize()
    for name in ("iterations", "flags", "flips_total", "bit_errors", "z_bits"):
        a = getattr(whole, name).cpu().numpy()
        b = np.concatenate([getattr(r, name).cpu().numpy() for r in parts])
        assert np.array_equal(a, b), name
    assert np.array_equal(whole.counters.cpu().numpy(), sum(r.counters.cpu().numpy() for r in parts))
    assert np.array_equal(whole.iter_hist.cpu().numpy(), sum(r.iter_hist.cpu().numpy() for r in parts))
