"""Benchmark: FWBF decoded information Gbit/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
EG(1023,781) type-I cyclic EG-LDPC, all-zero codeword, BPSK/AWGN at Eb/N0 =
4.0 dB (middle of the 3.0-5.0 sweep), float32 y, FWBF p = 31, alpha = 0.2,
K_max = 100, 2^20 frames per GPU resident in HBM (4.29 GB > L2: no flush
needed).  One step = one decode of the whole batch through the C ABI (plus
the NCCL all-reduce of the error/iteration counters when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU); frames shard with no data
exchange (weak scaling: 2^20 frames per GPU).  `--impl reference` times the
CPU decoder (the oracle port of the reference's numpy loop) on this host.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

K_INFO = {"eg5": 781, "eg4": 175, "eg6": 3367, "gal504": 252, "qc4x32": 14339}
CODE_NAMES = {"eg5": "EG(1023,781)", "eg4": "EG(255,175)", "eg6": "EG(4095,3367)",
              "gal504": "Gallager(3,6) N=504", "qc4x32": "QC(4,32) N=16384"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--code", default="eg5")
    ap.add_argument("--frames", type=int, default=1 << 20)
    ap.add_argument("--ebn0", type=float, default=4.0)
    ap.add_argument("--p", type=int, default=31)
    ap.add_argument("--kmax", type=int, default=100)
    ap.add_argument("--alpha", type=float, default=0.2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="bounded CPU sample (seconds of work) for the cpu_baseline leg")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: total timed CPU work over the K steps")
    ap.add_argument("--ref-1worker-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=1 << 14)
    return ap.parse_args()


# --------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------- CPU reference arm
#
# The reference decoder is pure Python + numpy (fwbf 0.1.0).  It is installed
# unmodified into baseline/_ref (pip --target) and run
# through its own public Monte Carlo entry point, harness.run_point
# (/root/reference/pkg/src/fwbf/harness.py:118-173), on the bench workload:
# same code, decoder, p, alpha, K_max and Eb/N0, the reference's own channel
# (float64 y), `workers` = all host cores, target_word_errors huge so the run
# is a fixed number of frames.  The code is built once, outside the timed
# region; the rate is passed so run_point skips its GF(2) rank.  If
# baseline/_ref is missing, the oracle port (oracle/wbf_oracle.py) stands in
# and `kind` says "port".

def _host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def _ref_fwbf():
    """The installed reference package (baseline/_ref), or None."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "fwbf")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import fwbf  # noqa: F401
    except Exception:
        return None
    if not os.path.abspath(fwbf.__file__).startswith(path):
        return None
    return fwbf


class CpuArm:
    """The reference's own run_point (or the oracle port) on this host's cores."""

    def __init__(self, a, workers: int):
        self.a, self.workers = a, workers
        self.k = K_INFO[a.code]
        self.fw = _ref_fwbf()
        from tests.golden.codebook import build_code
        if self.fw is not None:
            self.kind = "reference"
            if a.code == "eg5":
                self.h = self.fw.eg_ldpc_construct(5)          # the reference's own constructor
            else:
                hh = build_code(a.code)
                self.h = self.fw.ParityCheckMatrix(hh.row_adj, hh.n_cols)
        else:
            self.kind = "port"
            self.h = build_code(a.code)

    def run(self, frames: int):
        """Decode `frames` frames; returns (frames, seconds, mean iterations)."""
        a = self.a
        if self.fw is not None:
            fw = self.fw
            cfg = fw.DecoderConfig(alpha=a.alpha, k_max=a.kmax, block_len_p=a.p)
            ec = fw.ExperimentConfig(h=self.h, decoder="fwbf", decoder_cfg=cfg, ebn0_db=(a.ebn0,),
                                     rate=self.k / self.h.n_cols, target_word_errors=1 << 62,
                                     max_frames=frames, master_seed=a.seed, workers=self.workers)
            t0 = time.perf_counter()
            st = fw.run_point(ec, a.ebn0)
            return st.frames, time.perf_counter() - t0, st.mean_iters
        return port_decode_rate(a, frames, self.workers)

    def calibrated_frames(self, seconds: float) -> int:
        """Frames for about `seconds` of work (whole 128-frame batches per worker)."""
        unit = 128 * self.workers
        n, dt, _ = self.run(unit)
        fps = n / max(dt, 1e-6)
        return max(unit, int(fps * seconds / unit + 0.5) * unit)

    def sample_text(self, frames: int) -> str:
        a = self.a
        if self.kind == "reference":
            return (f"{frames} frames per run of the bench workload through the installed reference's own "
                    f"fwbf.harness.run_point (baseline/_ref, unmodified; reference channel, float64 y), "
                    f"workers={self.workers}")
        return (f"{frames} seeded frames of the bench workload through oracle/wbf_oracle.py (numpy "
                f"restatement of the reference decode loop), {self.workers}-process pool")


def _port_worker(args):
    code, ebn0, p, kmax, alpha, seed, start, count = args
    import numpy as np
    from oracle import wbf_oracle as O
    from tests.golden.codebook import build_code, code_rate
    g = O.Graph.of(build_code(code))
    sigma = O.ebn0_to_sigma(ebn0, code_rate(code))
    its = 0
    for i in range(start, start + count):
        y = O.channel_frame(np.zeros(g.n, np.uint8), sigma, seed, i)
        its += O.decode(g, y, "fwbf", alpha=alpha, k_max=kmax, p=p).iterations
    return count, its


def port_decode_rate(a, frames: int, cores: int):
    """Fallback when baseline/_ref is absent: the oracle port over `frames` frames."""
    from multiprocessing import get_context
    chunk = 128
    jobs = [(a.code, a.ebn0, a.p, a.kmax, a.alpha, a.seed, s, min(chunk, frames - s))
            for s in range(0, frames, chunk)]
    t0 = time.perf_counter()
    if cores == 1:
        res = [_port_worker(j) for j in jobs]
    else:
        with get_context("fork").Pool(cores) as pool:
            res = pool.map(_port_worker, jobs)
    dt = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    return n, dt, sum(r[1] for r in res) / max(1, n)


def run_reference(a, rank: int):
    """--impl reference: rank 0 times the reference CPU decoder; other ranks exit."""
    if rank != 0:
        return
    cores = _host_cores()
    arm = CpuArm(a, cores)
    # per-step sample: the whole timed run takes about ref_seconds (>= 30 s of
    # work), split over the K steps in whole batches per worker
    step_s = max(2.0, a.ref_seconds / max(1, a.steps))
    frames = arm.calibrated_frames(step_s)   # also the warm-up (pool start, imports)
    times, its, nfr = [], [], 0
    for _ in range(a.steps):
        n, dt, mi = arm.run(frames)
        times.append(dt)
        its.append(mi)
        nfr += n
    t = sum(times)
    value = nfr * arm.k / t / 1e9
    one = CpuArm(a, 1)
    f1 = one.calibrated_frames(a.ref_1worker_seconds)
    n1, dt1, _ = one.run(f1)
    line = {
        "impl": "reference", "metric": "FWBF decoded info Gbit/s", "value": value, "unit": "Gbit/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * t / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference channel, seeded)",
        "config": config_dict(a, mean_iters=statistics.mean(its)),
        "cpu_baseline": {"value": value, "unit": "Gbit/s", "cores": cores, "kind": arm.kind,
                         "sample": arm.sample_text(frames) + f"; {a.steps} runs, {t:.1f} s timed in total"},
        "cpu_1worker": {"value": n1 * arm.k / dt1 / 1e9, "unit": "Gbit/s", "cores": 1, "frames": n1,
                        "seconds": dt1},
        "e2e": {"value": value, "unit": "Gbit/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(a, **extra):
    d = {"workload": f"{CODE_NAMES[a.code]} FWBF p={a.p} alpha={a.alpha} K_max={a.kmax} "
                     f"Eb/N0={a.ebn0} dB, all-zero codeword, float32 y",
         "code": CODE_NAMES[a.code], "frames_per_gpu": a.frames, "p": a.p, "k_max": a.kmax,
         "alpha": a.alpha, "ebn0_db": a.ebn0, "stall": "flip-global-max",
         "l2": "inputs larger than L2 (frames*4 KiB >> 126 MB); no flush",
         "parallelism": f"frames sharded over {a.gpus} GPU(s), NCCL all-reduce of counters"}
    d.update(extra)
    return d


# ------------------------------------------------------------------ our arm

def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1206_3362_b200 import DecoderConfig, _native as nat
    from paper_1206_3362_b200.decoders import device_code, make_params, BatchResult, _outputs
    from paper_1206_3362_b200.sharding import reduce_counters
    from tests.golden.codebook import build_code, code_rate
    import ctypes as C

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    h = build_code(a.code)
    n = h.n_cols
    kinfo = K_INFO[a.code]
    sigma = float(math.sqrt(1.0 / (2.0 * code_rate(a.code) * 10.0 ** (a.ebn0 / 10.0))))
    ld = (n + 3) // 4 * 4
    B = a.frames
    # synthetic channel output resident in HBM (seeded per rank)
    g = torch.Generator(device=dev).manual_seed(a.seed * 1000003 + rank)
    y = torch.empty((B, ld), dtype=torch.float32, device=dev)
    for s in range(0, B, 1 << 16):
        e = min(B, s + (1 << 16))
        y[s:e].normal_(generator=g).mul_(sigma).add_(1.0)
    dc = device_code(h, local)
    cfg = DecoderConfig(alpha=a.alpha, k_max=a.kmax, block_len_p=a.p)
    prm = make_params(cfg, "fwbf")
    L = nat.lib()
    zw = (n + 31) // 32
    res = BatchResult(n=n, z_bits=torch.zeros((B, zw), dtype=torch.int32, device=dev),
                      iterations=torch.zeros(B, dtype=torch.int32, device=dev),
                      flags=torch.zeros(B, dtype=torch.uint8, device=dev),
                      flips_total=torch.zeros(B, dtype=torch.int32, device=dev),
                      bit_errors=torch.zeros(B, dtype=torch.int32, device=dev),
                      counters=torch.zeros(nat.NCOUNTERS, dtype=torch.int64, device=dev))
    res.iter_hist = torch.zeros(a.kmax + 1, dtype=torch.int64, device=dev)
    out = _outputs(res)
    stream = torch.cuda.current_stream(dev)

    def step():
        res.counters.zero_()
        res.iter_hist.zero_()
        nat.check(L.fwbf_decode_f32(dc.handle, C.byref(prm), C.c_void_p(y.data_ptr()), B, ld,
                                    C.byref(out), C.c_void_p(stream.cuda_stream)), "decode")
        reduce_counters(res.counters)
        reduce_counters(res.iter_hist)

    for _ in range(a.warmup):
        step()
    launch_kernels = nat.last_kernel()
    torch.cuda.synchronize()
    dc.filter_stats(reset=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    fstats = dc.filter_stats(reset=True)   # exact resolutions of the filtered metric, timed steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    cnt = res.counters.cpu().numpy()   # last step, all ranks (all-reduced)
    frames_all = int(cnt[nat.CNT_FRAMES])
    mean_iters = cnt[nat.CNT_ITER_SUM] / frames_all
    value = world * B * a.steps * kinfo / (ms_max / 1e3) / 1e9
    ms_step = ms_max / a.steps

    # ---- end-to-end through the host-buffer C ABI (pinned host y -> results in host memory)
    e2e = None
    if not a.no_e2e:
        yh = torch.empty((B, ld), dtype=torch.float32, pin_memory=True)
        yh.copy_(y)
        zh = torch.empty((B, zw), dtype=torch.int32, pin_memory=True)
        ih = torch.empty(B, dtype=torch.int32, pin_memory=True)
        fh = torch.empty(B, dtype=torch.uint8, pin_memory=True)
        ch = np.zeros(nat.NCOUNTERS, np.int64)

        def e2e_step():
            nat.check(L.fwbf_decode_host_f32(
                dc.handle, C.byref(prm), C.c_void_p(yh.data_ptr()), B, ld,
                C.c_void_p(zh.data_ptr()), zw, C.c_void_p(ih.data_ptr()), C.c_void_p(fh.data_ptr()),
                ch.ctypes.data_as(C.c_void_p), a.e2e_chunk), "decode_host")

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        te = time.perf_counter() - t0
        tt = torch.tensor([te], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        te = float(tt.item())
        # what the PCIe link alone allows: the same pinned buffer copied to the device, nothing else running
        torch.cuda.synchronize()
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record()
        y.copy_(yh, non_blocking=True)
        pe1.record()
        torch.cuda.synchronize()
        h2d_gbs = B * ld * 4 / (pe0.elapsed_time(pe1) / 1e3) / 1e9
        e2e = {"value": world * B * a.steps * kinfo / te / 1e9, "unit": "Gbit/s",
               "h2d_link_GBps": h2d_gbs,
               "h2d_link_bound": world * h2d_gbs * 1e9 / (ld * 4) * kinfo / 1e9,
               "h2d_bytes_per_step": B * ld * 4,
               "d2h_bytes_per_step": B * (zw * 4 + 4 + 1) + nat.NCOUNTERS * 8,
               "path": ("fwbf_decode_host_f32 (pinned host y; chunked H2D / decode / D2H on 5 streams ordered by events: "
                        "consecutive chunks' decode kernels on alternating streams, so a chunk's drain overlaps the next chunk)"),
               "chunk_frames": a.e2e_chunk}

    if rank == 0:
        props = torch.cuda.get_device_properties(dev)
        sms = props.multi_processor_count
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
        except OSError:
            pass
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        csum = clk.summary()
        max_mhz = csum.get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
        bytes_frame = 4 * n + 4 * zw + 8
        launch_ms = ms_step  # one decode launch per step on this stream
        achieved = B * bytes_frame / (launch_ms / 1e3) / 1e9
        # ncu DRAM bytes of one decode launch (profiles/roofline_traffic.json,
        # captured on a smaller launch of the same workload) scaled per frame
        # to this run's launch of B frames, like `achieved`
        traffic, traffic_src, trf = None, None, {}
        try:
            tr = json.load(open(os.path.join(REPO, "profiles", "roofline_traffic.json"))).get(a.code, {})
            trf = tr
            if tr.get("dram_bytes_per_frame"):
                traffic = tr["dram_bytes_per_frame"] * B
                traffic_src = (f"{tr.get('source')}: {tr['dram_bytes_per_frame']:.0f} B/frame measured on a "
                               f"{tr.get('frames_per_launch')}-frame launch, x {B} frames")
        except OSError:
            pass
        edges = h.n_edges
        edge_visits = B * edges * (1.0 + mean_iters)
        ev_rate = edge_visits / (launch_ms / 1e3)
        dadd_peak = sms * 64 * max_mhz * 1e6
        smem_peak = sms * 128 * max_mhz * 1e6
        # filtered gather (FWBF on split-path frames).  Q16 (the default): one
        # 4-byte LDS brings the int16 quantised signed minima of two columns, two
        # IDP.2A add them -- 2 B of shared memory per edge visit, so 128 B/clk/SM
        # caps the gather at 64 visits/clk/SM.  FWBF_Q16=0: the float32 gather
        # (8-byte LDS + FADD2), 4 B per edge visit, 32 visits/clk/SM.
        q16 = os.environ.get("FWBF_Q16", "1") != "0"
        gather_bytes = 2 if q16 else 4
        gather_bound = sms * (128.0 / gather_bytes) * max_mhz * 1e6
        block_decisions = B * a.steps * ((n + a.p - 1) // a.p) * mean_iters
        line = {
            "metric": "FWBF decoded info Gbit/s", "value": value, "unit": "Gbit/s",
            "n_gpus": world, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded AWGN, all-zero codeword)",
            "config": config_dict(a, mean_iters=float(mean_iters),
                                  fer=float(cnt[nat.CNT_WORD_ERRORS] / frames_all),
                                  ber=float(cnt[nat.CNT_BIT_ERRORS] / (frames_all * n)),
                                  ordered_path_frames=int(cnt[nat.CNT_ORDERED_FRAMES]),
                                  iter_hist=[int(v) for v in res.iter_hist.cpu().tolist()],
                                  frames_per_s=world * B / (ms_step / 1e3)),
            # The binding roofline: the path is issue-bound, not
            # HBM-bound.  achieved = edge visits E (1 + I) per frame x frames/s
            # over the decode launches (CUDA events on the launch stream);
            # peak = one fp64 add per lane per clock = SMs x 64 x clock.  The
            # ncu issue-slot and shared-pipe utilisations of the same kernel
            # (profiles/roofline_traffic.json) ride along; HBM is a sub-record.
            "roofline": {"bound": "issue", "resource": "fp64-lane edge visits (one add per lane per clock)",
                         "achieved": ev_rate, "peak": dadd_peak, "unit": "edge-visits/s",
                         "frac": ev_rate / dadd_peak,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "edge_visits_per_frame": edges * (1.0 + mean_iters),
                         "ncu_issue_active_pct": trf.get("ncu_issue_active_pct"),
                         "ncu_smem_pipe_pct": trf.get("ncu_smem_pipe_pct"),
                         "ncu_source": trf.get("ncu_source"),
                         "clock_mhz_for_peaks": max_mhz,
                         "gather_bound": {
                             "resource": ("shared memory: filtered metric gather, int16 quantised minima (one 4-byte "
                                          "LDS + two IDP.2A per two edge visits; 2 B/edge at 128 B/clk/SM = 64 edge "
                                          "visits/clk/SM)") if q16 else
                                         ("shared memory: filtered metric gather (one 8-byte LDS + one FADD2 "
                                          "per two edge visits; 4 B/edge at 128 B/clk/SM = 32 edge visits/clk/SM)"),
                             "peak": gather_bound, "frac": ev_rate / gather_bound,
                             "smem_gather_bytes_per_edge": gather_bytes,
                             "smem_gather_bytes_per_s": gather_bytes * ev_rate,
                             "smem_peak_GBps": smem_peak / 1e9},
                         "filter": {"exact_block_decisions": fstats[0],
                                    "exact_fraction": fstats[0] / max(1.0, block_decisions),
                                    "exact_stall_argmaxes": fstats[1]},
                         "hbm": {"achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                                 "frac": achieved / hbm_peak, "bytes_per_frame": bytes_frame,
                                 "traffic": traffic,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}},
            "e2e": e2e,
            # per step: the filtered circulant kernel + decode_kernel over the
            # frames it deferred (2 launches when the circulant kernel applies)
            "gpu_launches": a.steps * (2 if launch_kernels.startswith("cdecode+") else 1),
            "decode_kernels": launch_kernels,
            "clocks": csum,
        }
        if not a.no_cpu_baseline and world == 1:
            cores = _host_cores()
            arm = CpuArm(a, cores)
            nf0 = arm.calibrated_frames(a.cpu_seconds)
            nf, dt, _ = arm.run(nf0)
            line["cpu_baseline"] = {"value": nf * kinfo / dt / 1e9, "unit": "Gbit/s", "cores": cores,
                                    "kind": arm.kind, "sample": arm.sample_text(nf) + f", {dt:.1f} s"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
