"""N>1 path on CPU: world_size-2 gloo ranks shard frames by global index and
all-reduce the int64 counters; totals must equal the single-process ones."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import wbf_oracle as O
from paper_1206_3362_b200.sharding import frame_shard, reduce_counters
from tests.golden.codebook import build_code, code_rate


def _counters(h, start, n, sigma):
    g = O.Graph.of(h)
    c = np.zeros(g.n, np.uint8)
    out = np.zeros(6, np.int64)
    if n:
        res = O.run_batch(g, "fwbf", sigma, 1, start, n, p=16, k_max=30)
        out[:] = res
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = build_code("eg4")
    sigma = O.ebn0_to_sigma(3.0, code_rate("eg4"))
    s, n = frame_shard(0, 40, rank, world)
    t = torch.from_numpy(_counters(h, s, n, sigma))
    reduce_counters(t)
    if rank == 0:
        q.put(t.numpy().tolist())
    dist.destroy_process_group()


def test_gloo_world2_counter_allreduce():
    h = build_code("eg4")
    sigma = O.ebn0_to_sigma(3.0, code_rate("eg4"))
    ref = _counters(h, 0, 40, sigma).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert got == ref


# ---- distributed run_point: batch sharding + per-batch table all-reduce ----

def mock_decode(start, count):
    """Deterministic per-frame stand-in for the CUDA decoder: per-128-batch sums
    [frames, bit_err, word_err, iters, flips, stalls] of frames [start, start+count),
    a function of the global frame index only (like the real decoder)."""
    f = np.arange(start, start + count, dtype=np.int64)
    we = ((f * 2654435761) % 97 < 3).astype(np.int64)
    rows = np.stack([np.ones_like(f), we * (1 + f % 5), we, 1 + f % 13, f % 7, (f % 211 == 0).astype(np.int64)], 1)
    nb = -(-count // 128)
    pad = nb * 128 - count
    if pad:
        rows = np.concatenate([rows, np.zeros((pad, 6), np.int64)])
    return rows.reshape(nb, 128, 6).sum(1)


def _point_cfg():
    from paper_1206_3362_b200 import DecoderConfig
    from paper_1206_3362_b200.harness import ExperimentConfig
    return ExperimentConfig(h=build_code("eg4"), decoder="fwbf", decoder_cfg=DecoderConfig(block_len_p=16),
                            ebn0_db=(3.0,), rate=175 / 255, target_word_errors=40, max_frames=20000,
                            chunk_frames=1000)


def _point_worker(rank, world, port, q):
    from paper_1206_3362_b200.harness import run_point
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = run_point(_point_cfg(), 3.0, _decode=mock_decode)
    q.put((rank, (st.frames, st.bit_errors, st.word_errors, st.mean_iters, st.stalls, st.capped)))
    dist.destroy_process_group()


def test_gloo_world2_run_point_matches_single_process():
    from paper_1206_3362_b200.harness import run_point
    st = run_point(_point_cfg(), 3.0, _decode=mock_decode)
    ref = (st.frames, st.bit_errors, st.word_errors, st.mean_iters, st.stalls, st.capped)
    assert st.frames % 128 == 0 and st.word_errors >= 40  # stopped by the rule, at a batch boundary
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_point_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert got[0] == ref and got[1] == ref
