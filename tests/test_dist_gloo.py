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
