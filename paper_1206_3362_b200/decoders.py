"""Drop-in decoder entry points backed by the CUDA library.

Mirrors the public surface of the reference module
`/root/reference/pkg/src/fwbf/decoders.py`:

  DecoderConfig            decoders.py:32-61  (same fields, same ValueErrors)
  DecodeOutcome            decoders.py:124-135
  DecodeState              decoders.py:111-121
  decode_imwbf             decoders.py:232-235
  decode_mlp_wbf           decoders.py:238-247
  decode_fwbf              decoders.py:250-259

and adds the batched seam `decode_batch(h, Y, cfg, algorithm)` that the
per-frame functions are thin wrappers of.  Every decode runs on the GPU
through libfwbf_b200.so; there is no CPU decoder in this package.

`weight_mode` ("imwbf" Eq.(1) exclude-self weights, or "mwbf" include-self
minimum) extends DecoderConfig so WBF (mwbf, alpha=0) and MWBF run through the
same loop; the default reproduces the reference exactly.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _native as nat

STALL_POLICIES = ("terminate", "flip-global-max")
WEIGHT_MODES = ("imwbf", "mwbf")


@dataclass(frozen=True)
class DecoderConfig:
    """Knobs shared by the decoder family (reference decoders.py:32-61)."""

    alpha: float = 0.2
    k_max: int = 10
    lam: int = 1
    block_len_p: Optional[int] = None
    stall_policy: str = "flip-global-max"
    mlp_threshold: bool = True
    weight_mode: str = "imwbf"

    def __post_init__(self):
        if self.alpha < 0:
            raise ValueError("alpha must be nonnegative")
        if self.k_max < 1:
            raise ValueError("k_max must be >= 1")
        if self.lam < 1:
            raise ValueError("lam must be >= 1")
        if self.block_len_p is not None and self.block_len_p < 1:
            raise ValueError("block_len_p must be >= 1")
        if self.stall_policy not in STALL_POLICIES:
            raise ValueError(f"stall_policy must be one of {STALL_POLICIES}")
        if self.weight_mode not in WEIGHT_MODES:
            raise ValueError(f"weight_mode must be one of {WEIGHT_MODES}")


@dataclass
class DecodeState:
    """Snapshot of the decode loop at the top of one iteration (decoders.py:111-121)."""

    z: np.ndarray
    syndrome: np.ndarray
    iteration: int

    @property
    def syndrome_weight(self) -> int:
        return int(np.count_nonzero(self.syndrome))


@dataclass
class DecodeOutcome:
    """Per-frame result (decoders.py:124-135)."""

    z_final: np.ndarray
    iterations: int
    converged: bool
    flip_log: List[List[int]]
    stalled: bool
    trace: Optional[List[DecodeState]] = field(default=None, repr=False)

    @property
    def flips_total(self) -> int:
        return sum(len(f) for f in self.flip_log)


# ---------------------------------------------------------------------------
# Device code handles
# ---------------------------------------------------------------------------

class DeviceCode:
    """H resident on one device (owns the C handle).

    Built from any matrix exposing ``row_adj`` and ``n_cols`` -- this package's
    ParityCheckMatrix or the reference's own (matrix.py:22-58).  Circulant
    matrices are passed as their first row (index arithmetic on the device)."""

    def __init__(self, h, device: int = 0):
        from .codes import detect_structure, ParityCheckMatrix
        L = nat.lib()
        self.n = int(h.n_cols)
        self.m = len(h.row_adj)
        self.device = int(device)
        rows = [np.asarray(r, dtype=np.int64) for r in h.row_adj]
        row_ptr = np.zeros(self.m + 1, np.int32)
        np.cumsum([r.size for r in rows], out=row_ptr[1:])
        row_idx = (np.concatenate(rows) if rows else np.zeros(0, np.int64)).astype(np.int32)
        self.n_edges = int(row_idx.size)
        pcm = h if isinstance(h, ParityCheckMatrix) else ParityCheckMatrix(rows, self.n)
        st = detect_structure(pcm)
        self.structure = st.kind
        self._keep = [row_ptr, row_idx]
        desc = nat.CodeDesc()
        desc.n_cols = self.n
        desc.n_rows = self.m
        desc.row_ptr = row_ptr.ctypes.data_as(C.POINTER(C.c_int32))
        desc.row_idx = row_idx.ctypes.data_as(C.POINTER(C.c_int32))
        if st.kind == "circulant" and st.offsets.size <= 64:
            offs = st.offsets.astype(np.int32)
            self._keep.append(offs)
            desc.circulant = 1
            desc.n_offsets = int(offs.size)
            desc.offsets = offs.ctypes.data_as(C.POINTER(C.c_int32))
        self.row_weights = np.diff(row_ptr)
        handle = C.c_void_p()
        nat.check(L.fwbf_code_create(C.byref(desc), self.device, C.byref(handle)), "code_create")
        self.handle = handle
        self._fin = weakref.finalize(self, L.fwbf_code_destroy, handle)

    def close(self):
        self._fin()

    def filter_stats(self, reset: bool = False) -> Tuple[int, int]:
        """(block argmaxes, stall argmaxes) the filtered FWBF metric resolved with
        exact column sums in this code's launches so far (diagnostic)."""
        out = (C.c_int64 * 2)()
        nat.check(nat.lib().fwbf_filter_stats(self.handle, out, 1 if reset else 0), "filter_stats")
        return int(out[0]), int(out[1])


_CODES: Dict[Tuple[int, int], DeviceCode] = {}


def device_code(h, device: int = 0) -> DeviceCode:
    """Cached DeviceCode for (h, device); dropped when h is garbage collected."""
    if isinstance(h, DeviceCode):
        return h
    key = (id(h), int(device))
    dc = _CODES.get(key)
    if dc is None:
        dc = DeviceCode(h, device)
        _CODES[key] = dc
        try:
            weakref.finalize(h, _CODES.pop, key, None)
        except TypeError:
            # not weak-referenceable: hold h so its id cannot be reused by
            # another matrix while the cached handle exists
            dc._owner = h
    return dc


def make_params(cfg: DecoderConfig, algorithm: str, force_ordered=False) -> nat.Params:
    if algorithm not in nat.ALG:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    p = nat.Params()
    p.algorithm = nat.ALG[algorithm]
    p.weight_mode = nat.WEIGHTS[getattr(cfg, "weight_mode", "imwbf")]
    p.alpha = float(cfg.alpha)
    p.k_max = int(cfg.k_max)
    p.lam = int(cfg.lam)
    p.block_len_p = int(cfg.block_len_p) if cfg.block_len_p is not None else 0
    p.stall = nat.STALL[cfg.stall_policy]
    p.mlp_threshold = 1 if cfg.mlp_threshold else 0
    p.force_ordered = int(force_ordered)  # bit flags: 1 ordered path; 2 no split-fp32 path; 4 no filtered metric
    return p


# ---------------------------------------------------------------------------
# Batched decode
# ---------------------------------------------------------------------------

@dataclass
class BatchResult:
    """Per-frame device outputs of one decode_batch call (torch tensors)."""

    n: int
    z_bits: "object"            # int32 [B, ceil(n/32)] (bit n%32 of word n//32)
    iterations: "object"        # int32 [B]
    flags: "object"             # uint8 [B]
    flips_total: "object"       # int32 [B]
    bit_errors: "object"        # int32 [B]
    counters: "object"          # int64 [NCOUNTERS]
    fliplog: "object" = None    # int32 [B, stride]
    fliplog_counts: "object" = None  # int32 [B, k_max]
    iter_hist: "object" = None  # int64 [k_max + 1]: frames that stopped after k iterations

    def z(self) -> np.ndarray:
        w = self.z_bits.cpu().numpy().astype(np.uint32)
        bits = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")
        return bits[:, :self.n]

    @property
    def converged(self) -> np.ndarray:
        return (self.flags.cpu().numpy() & nat.FLAG_CONVERGED) != 0

    @property
    def stalled(self) -> np.ndarray:
        return (self.flags.cpu().numpy() & nat.FLAG_STALLED) != 0

    def flip_logs(self) -> List[List[List[int]]]:
        if self.fliplog is None:
            raise ValueError("decode_batch was called without flip_log=True")
        cnt = self.fliplog_counts.cpu().numpy()
        log = self.fliplog.cpu().numpy()
        its = self.iterations.cpu().numpy()
        out = []
        for f in range(its.size):
            frame, pos = [], 0
            for k in range(int(its[f])):
                c = int(cnt[f, k])
                frame.append(log[f, pos:pos + c].tolist())
                pos += c
            out.append(frame)
        return out


def _torch():
    import torch
    return torch


def _outputs(res: BatchResult, stride: int = 0, codeword_t=None) -> nat.Outputs:
    o = nat.Outputs()
    o.z_bits = res.z_bits.data_ptr()
    o.z_ld = res.z_bits.shape[1]
    o.iterations = res.iterations.data_ptr()
    o.flags = res.flags.data_ptr()
    o.flips_total = res.flips_total.data_ptr()
    o.bit_errors = res.bit_errors.data_ptr()
    o.counters = res.counters.data_ptr()
    if res.iter_hist is not None:
        o.iter_hist = res.iter_hist.data_ptr()
    if res.fliplog is not None:
        o.fliplog = res.fliplog.data_ptr()
        o.fliplog_counts = res.fliplog_counts.data_ptr()
        o.fliplog_stride = stride
    if codeword_t is not None:
        o.codeword_bits = codeword_t.data_ptr()
    return o


def pack_bits(c: np.ndarray, n: int) -> np.ndarray:
    """uint8 bit vector -> little-endian uint32 words (layout of z_bits)."""
    c = np.asarray(c, dtype=np.uint8).reshape(-1)
    if c.shape != (n,):
        raise ValueError(f"codeword must have length {n}")
    words = (n + 31) // 32
    buf = np.zeros(words * 32, np.uint8)
    buf[:n] = c
    return np.packbits(buf, bitorder="little").view(np.uint32)


def _launch_stream(dev, stream, tensors):
    """The stream the C call is enqueued on.  A caller-supplied stream first
    waits for the current stream (where the inputs were copied and the outputs
    zero-filled), and every tensor is recorded on it so the caching allocator
    keeps the memory until that stream has consumed it."""
    torch = _torch()
    cur = torch.cuda.current_stream(dev)
    if stream is None or stream == cur:
        return cur
    stream.wait_stream(cur)
    for t in tensors:
        if t is not None:
            t.record_stream(stream)
    return stream


def _result_tensors(res: "BatchResult"):
    return [res.z_bits, res.iterations, res.flags, res.flips_total, res.bit_errors, res.counters,
            res.fliplog, res.fliplog_counts, res.iter_hist, getattr(res, "batch_word_err", None),
            getattr(res, "y", None)]


def _new_result(torch, n, B, zw, k_max, kw, batches=0):
    """Output tensors of one decode.  Per-frame outputs are written for every
    frame by the kernels, so they start uninitialised; the accumulated ones
    (counters, iteration histogram, per-batch word errors) are views of one
    zeroed allocation -- one memset instead of eight per call (small batches
    are launch-bound)."""
    nacc = nat.NCOUNTERS + k_max + 1 + (batches + 1) // 2
    acc = torch.zeros(nacc, dtype=torch.int64, **kw)
    res = BatchResult(
        n=n,
        z_bits=torch.empty((B, zw), dtype=torch.int32, **kw),
        iterations=torch.empty(B, dtype=torch.int32, **kw),
        flags=torch.empty(B, dtype=torch.uint8, **kw),
        flips_total=torch.empty(B, dtype=torch.int32, **kw),
        bit_errors=torch.empty(B, dtype=torch.int32, **kw),
        counters=acc[:nat.NCOUNTERS],
        iter_hist=acc[nat.NCOUNTERS:nat.NCOUNTERS + k_max + 1])
    if batches:
        res.batch_word_err = acc[nat.NCOUNTERS + k_max + 1:].view(torch.int32)[:batches]
    return res


def decode_batch(h, y, cfg: DecoderConfig, algorithm: str = "fwbf", *, flip_log: bool = False,
                 codeword=None, device=None, force_ordered: bool = False, stream=None) -> BatchResult:
    """Decode a batch of frames Y[B, ld>=N] (float32 or float64; torch or numpy).

    Same semantics per frame as the reference loop (decoders.py:189-229).  A
    float32 Y is decoded as its exact float64 upcast, exactly like the
    reference does with float32 input."""
    torch = _torch()
    if algorithm == "fwbf" and cfg.block_len_p is None:
        raise ValueError("block_len_p is required for block-parallel decoding")
    if not isinstance(y, torch.Tensor):
        arr = np.asarray(y)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        y = torch.from_numpy(np.ascontiguousarray(arr))
    if y.dim() == 1:
        y = y.unsqueeze(0)
    if y.dtype not in (torch.float32, torch.float64):
        y = y.to(torch.float64)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    if dev.type != "cuda":
        raise ValueError("decode_batch needs a CUDA device")
    y = y.to(dev)
    if y.stride(1) != 1:
        y = y.contiguous()
    with torch.cuda.device(dev):
        dc = device_code(h, dev.index if dev.index is not None else 0)
    if y.shape[1] < dc.n:
        raise ValueError(f"expected a length-{dc.n} frame")
    if y.shape[1] != dc.n and y.stride(0) != y.shape[1]:
        y = y.contiguous()
    B, ld = int(y.shape[0]), int(y.stride(0))
    if B <= 1:
        ld = int(y.shape[1])  # a single row may carry any (even zero) row stride
    p = make_params(cfg, algorithm, force_ordered)
    L = nat.lib()
    zw = (dc.n + 31) // 32
    kw = dict(device=dev)
    res = _new_result(torch, dc.n, B, zw, cfg.k_max, kw)
    stride = 0
    if flip_log:
        maxf = int(L.fwbf_max_flips_per_iter(dc.handle, C.byref(p)))
        stride = max(1, cfg.k_max * maxf)
        res.fliplog = torch.full((B, stride), -1, dtype=torch.int32, **kw)
        res.fliplog_counts = torch.zeros((B, cfg.k_max), dtype=torch.int32, **kw)
    cw_t = None
    if codeword is not None:
        cw_t = torch.from_numpy(pack_bits(codeword, dc.n).view(np.int32)).to(dev)
    out = _outputs(res, stride, cw_t)
    st = _launch_stream(dev, stream, _result_tensors(res) + [y, cw_t])
    fn = L.fwbf_decode_f32 if y.dtype == torch.float32 else L.fwbf_decode_f64
    with torch.cuda.device(dev):
        nat.check(fn(dc.handle, C.byref(p), C.c_void_p(y.data_ptr()), B, ld, C.byref(out),
                     C.c_void_p(st.cuda_stream)), "decode")
    res._inputs = (y, cw_t)  # keep alive until the stream consumes them
    return res


def metric_batch(h, y, cfg: DecoderConfig = DecoderConfig(), algorithm: str = "fwbf", *,
                 force_ordered=False, device=None):
    """Stage view: the Eq.(1) metric of each frame's first iteration (the
    reference's ``all_metrics`` on the initial hard decisions with the weights
    of ``compute_weights``/``edge_weights``, decoders.py:80-103,148-153),
    computed by the decode kernel itself.  Returns (E float64 [B, N] torch
    tensor on the device, per-frame flags uint8)."""
    torch = _torch()
    if not isinstance(y, torch.Tensor):
        arr = np.asarray(y)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        y = torch.from_numpy(np.ascontiguousarray(arr))
    if y.dim() == 1:
        y = y.unsqueeze(0)
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    y = y.to(dev).contiguous()
    with torch.cuda.device(dev):
        dc = device_code(h, dev.index if dev.index is not None else 0)
    if y.shape[1] != dc.n:
        raise ValueError(f"expected a length-{dc.n} frame")
    B = int(y.shape[0])
    E = torch.empty((B, dc.n), dtype=torch.float64, device=dev)
    flags = torch.zeros(B, dtype=torch.uint8, device=dev)
    p = make_params(cfg, algorithm, force_ordered)
    L = nat.lib()
    fn = L.fwbf_metric_f32 if y.dtype == torch.float32 else L.fwbf_metric_f64
    st = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        nat.check(fn(dc.handle, C.byref(p), C.c_void_p(y.data_ptr()), B, dc.n, C.c_void_p(E.data_ptr()),
                     dc.n, C.c_void_p(flags.data_ptr()), C.c_void_p(st.cuda_stream)), "metric")
    return E, flags


def decode_awgn(h, cfg: DecoderConfig, algorithm: str, seed: int, first_frame: int, count: int,
                sigma: float, *, codeword=None, noise: str = "f64", flip_log: bool = False,
                device=None, force_ordered: bool = False, stream=None,
                batch_frames: int = 128, return_y: bool = False) -> BatchResult:
    """Decode frames [first_frame, first_frame + count) of the reference channel.

    The device draws y_n = (1 - 2 c_n) + sigma * g_n with g from numpy's
    Philox(key=seed, counter=frame << 128) + standard_normal stream
    (channel.py:29-50), i.e. the frames harness._run_batch would decode.
    noise="f64" keeps y in float64 (the reference's own values); "f32" rounds
    y to float32 first (the float32-input configs of BASELINE.json).
    Per-batch word errors (batch_frames frames each, harness.py:24) are
    returned in `res.batch_word_err`."""
    torch = _torch()
    if algorithm == "fwbf" and cfg.block_len_p is None:
        raise ValueError("block_len_p is required for block-parallel decoding")
    if seed < 0 or first_frame < 0:
        raise ValueError("seed and frame index must be nonnegative")
    if seed >= 1 << 64:
        # the device keys Philox with the low 64-bit key word only (channel.py:44)
        raise ValueError("seed must be below 2**64")
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        dc = device_code(h, dev.index if dev.index is not None else 0)
    p = make_params(cfg, algorithm, force_ordered)
    L = nat.lib()
    B = int(count)
    zw = (dc.n + 31) // 32
    kw = dict(device=dev)
    res = _new_result(torch, dc.n, B, zw, cfg.k_max, kw, batches=max(1, -(-B // batch_frames)))
    stride = 0
    if flip_log:
        maxf = int(L.fwbf_max_flips_per_iter(dc.handle, C.byref(p)))
        stride = max(1, cfg.k_max * maxf)
        res.fliplog = torch.full((B, stride), -1, dtype=torch.int32, **kw)
        res.fliplog_counts = torch.zeros((B, cfg.k_max), dtype=torch.int32, **kw)
    cw_t = None
    if codeword is not None:
        cw_t = torch.from_numpy(pack_bits(codeword, dc.n).view(np.int32)).to(dev)
    out = _outputs(res, stride, cw_t)
    out.batch_word_err = res.batch_word_err.data_ptr()
    out.batch_frames = int(batch_frames)
    res.y = None
    if return_y:  # the generated channel values (testing / inspection)
        res.y = torch.empty((B, dc.n), dtype=torch.float64 if noise == "f64" else torch.float32, **kw)
        out.y_out = res.y.data_ptr()
        out.y_out_ld = dc.n
    mode = {"f64": nat.NOISE_NUMPY_F64, "f32": nat.NOISE_NUMPY_F32}[noise]
    st = _launch_stream(dev, stream, _result_tensors(res) + [cw_t])
    with torch.cuda.device(dev):
        nat.check(L.fwbf_decode_awgn(dc.handle, C.byref(p), C.c_uint64(int(seed)), int(first_frame), B,
                                     float(sigma), mode, C.byref(out), C.c_void_p(st.cuda_stream)),
                  "decode_awgn")
    res._inputs = (cw_t,)
    return res


# ---------------------------------------------------------------------------
# Per-frame entry points (reference decoders.py:232-259)
# ---------------------------------------------------------------------------

def _trace_states(h, y: np.ndarray, log: List[List[int]]) -> List[DecodeState]:
    from .codes import ParityCheckMatrix
    pcm = h if isinstance(h, ParityCheckMatrix) else ParityCheckMatrix(h.row_adj, h.n_cols)
    z = (np.asarray(y, dtype=np.float64) < 0).astype(np.uint8)
    states = [DecodeState(z.copy(), pcm.syndrome(z), 0)]
    for k, flips in enumerate(log, start=1):
        if flips:
            z[np.asarray(flips, dtype=np.int64)] ^= 1
        states.append(DecodeState(z.copy(), pcm.syndrome(z), k))
    return states


def _decode_one(h, y, cfg: DecoderConfig, algorithm: str, trace: bool) -> DecodeOutcome:
    arr = np.asarray(y)
    n = int(h.n_cols)
    if arr.shape != (n,):
        raise ValueError(f"expected a length-{n} frame")
    if arr.dtype != np.float32:
        arr = arr.astype(np.float64)
    res = decode_batch(h, arr[None, :], cfg, algorithm, flip_log=True)
    log = res.flip_logs()[0]
    it = int(res.iterations.cpu()[0])
    fl = int(res.flags.cpu()[0])
    out = DecodeOutcome(z_final=res.z()[0].astype(np.uint8), iterations=it,
                        converged=bool(fl & nat.FLAG_CONVERGED), flip_log=log,
                        stalled=bool(fl & nat.FLAG_STALLED))
    if trace:
        out.trace = _trace_states(h, arr, log)
    return out


def decode_imwbf(h, y, cfg: DecoderConfig = DecoderConfig(), trace: bool = False) -> DecodeOutcome:
    """Flip the single largest-metric bit each iteration (ties: lowest index)."""
    return _decode_one(h, y, cfg, "imwbf", trace)


def decode_mlp_wbf(h, y, cfg: DecoderConfig = DecoderConfig(), trace: bool = False) -> DecodeOutcome:
    """Flip the bits holding the lam largest metrics each iteration."""
    if cfg.lam > h.n_cols:
        raise ValueError(f"lam={cfg.lam} exceeds block length {h.n_cols}")
    return _decode_one(h, y, cfg, "mlp", trace)


def decode_fwbf(h, y, cfg: DecoderConfig = DecoderConfig(block_len_p=1),
                trace: bool = False) -> DecodeOutcome:
    """Flip at most one bit per contiguous p-length block each iteration."""
    if cfg.block_len_p is None:
        raise ValueError("block_len_p is required for block-parallel decoding")
    return _decode_one(h, y, cfg, "fwbf", trace)
