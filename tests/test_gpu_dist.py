"""The N>1 path with the real CUDA decoder: two ranks under a
gloo process group, both on cuda:0 (the driver's boxes have one GPU; the ranks
never wait on each other's kernels), each decoding its shard of run_point's
batches with decode_awgn; the per-batch table is all-reduced and both ranks
must return the single-process statistics.  Also bench.py's counter
all-reduce over the decode counters."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _cfg():
    from paper_1206_3362_b200 import DecoderConfig
    from paper_1206_3362_b200.harness import ExperimentConfig
    from tests.golden.codebook import build_code
    return ExperimentConfig(h=build_code("eg5"), decoder="fwbf", decoder_cfg=DecoderConfig(block_len_p=31, k_max=100),
                            ebn0_db=(3.5,), target_word_errors=300, max_frames=40000, master_seed=4,
                            noise="f32", chunk_frames=4096)


def _stats(st):
    return (st.frames, st.bit_errors, st.word_errors, st.mean_iters, st.mean_flips, st.stalls, st.capped)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_1206_3362_b200.harness import run_point
    from paper_1206_3362_b200.sharding import frame_shard, reduce_counters
    from paper_1206_3362_b200.decoders import decode_awgn
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = _cfg()
    st = run_point(c, 3.5)
    # bench.py's step: each rank decodes its frame shard, counters all-reduced
    s0, n0 = frame_shard(0, 50000, rank, world)
    res = decode_awgn(c.h, c.decoder_cfg, "fwbf", 4, s0, n0, 0.54, noise="f32")
    cnt = res.counters.cpu()
    reduce_counters(cnt)
    q.put((rank, _stats(st), cnt.numpy().tolist()))
    dist.destroy_process_group()


def test_world2_run_point_and_counter_allreduce_with_cuda_decoder(cuda_device):
    from paper_1206_3362_b200.harness import run_point
    from paper_1206_3362_b200.decoders import decode_awgn
    c = _cfg()
    ref = _stats(run_point(c, 3.5))
    ref_cnt = decode_awgn(c.h, c.decoder_cfg, "fwbf", 4, 0, 50000, 0.54, noise="f32").counters.cpu().numpy().tolist()
    assert ref[2] >= 300 and ref[0] % 128 == 0          # stopped by the word-error rule
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, st, cnt = q.get(timeout=300)
        got[rank] = (st, cnt)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        assert got[r][0] == ref, (r, got[r][0], ref)
        assert got[r][1] == ref_cnt
