"""Stage-level decoder API on the device (reference decoders.py:64-167).

The decode kernel fuses every stage of the WBF loop; callers of the
reference's stage functions -- ``compute_weights``, ``WeightTable``,
``hard_decision``, ``all_metrics``, ``block_argmax``, ``bit_metric`` (exported
by the reference at ``__init__.py:13-15``) -- get them here under the same
names, signatures and ValueErrors, computed by the stage kernels of
libfwbf_b200.so (csrc/fwbf_stage.cu) in float64 exactly like numpy does.

Per-frame numpy inputs return numpy outputs (the reference's types); 2-D
inputs are treated as batches of frames, and CUDA tensors stay on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as nat


def _torch():
    import torch
    return torch


def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise nat.FwbfError("the stage kernels need a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _on_device(x, dtype):
    """(contiguous CUDA tensor of `dtype`, input was host data)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.to(_device())
        return t.to(dtype).contiguous(), False
    arr = np.ascontiguousarray(np.asarray(x))
    return torch.from_numpy(arr).to(_device()).to(dtype).contiguous(), True


def _out(t, host: bool):
    return t.cpu().numpy() if host else t


def _stream(t):
    return C.c_void_p(_torch().cuda.current_stream(t.device).cuda_stream)


def _code(h, t):
    from .decoders import device_code
    return device_code(h, t.device.index)


@dataclass
class WeightTable:
    """Per-check minima of |y| (decoders.py:64-84): the weight of edge (n, m)
    is min2[m] when n == argmin_col[m], else min1[m]."""

    min1: np.ndarray
    min2: np.ndarray
    argmin_col: np.ndarray

    def weight(self, m: int, n: int) -> float:
        return float(self.min2[m]) if n == self.argmin_col[m] else float(self.min1[m])

    def edge_weights(self, h) -> np.ndarray:
        """Weights in the row-major edge order of H (decoders.py:80-84)."""
        torch = _torch()
        m1, host = _on_device(self.min1, torch.float64)
        m2, _ = _on_device(self.min2, torch.float64)
        am, _ = _on_device(self.argmin_col, torch.int64)
        dc = _code(h, m1)
        batch = 1 if m1.dim() == 1 else int(m1.shape[0])
        shape = (dc.n_edges,) if m1.dim() == 1 else (batch, dc.n_edges)
        w = torch.empty(shape, dtype=torch.float64, device=m1.device)
        nat.check(nat.lib().fwbf_stage_edge_weights(dc.handle, m1.data_ptr(), m2.data_ptr(), am.data_ptr(),
                                                      batch, w.data_ptr(), _stream(m1)), "edge_weights")
        return _out(w, host)


def compute_weights(h, y) -> WeightTable:
    """Weight table of a frame (decoders.py:87-103); depends only on |y|.
    Raises ValueError for a check with fewer than 2 bits or a wrong length."""
    torch = _torch()
    rw = np.array([len(r) for r in h.row_adj])
    if len(rw) and int(rw.min()) < 2:
        raise ValueError("every check must contain at least 2 bits")
    yt, host = _on_device(y, torch.float64)
    n = int(h.n_cols)
    if yt.shape[-1] != n or yt.dim() not in (1, 2):
        raise ValueError(f"expected a length-{n} frame")
    dc = _code(h, yt)
    batch = 1 if yt.dim() == 1 else int(yt.shape[0])
    shape = (dc.m,) if yt.dim() == 1 else (batch, dc.m)
    kw = dict(device=yt.device)
    min1 = torch.empty(shape, dtype=torch.float64, **kw)
    min2 = torch.empty(shape, dtype=torch.float64, **kw)
    am = torch.empty(shape, dtype=torch.int64, **kw)
    nat.check(nat.lib().fwbf_stage_weights(dc.handle, yt.data_ptr(), batch, n, min1.data_ptr(), min2.data_ptr(),
                                             am.data_ptr(), None, _stream(yt)), "compute_weights")
    return WeightTable(min1=_out(min1, host), min2=_out(min2, host), argmin_col=_out(am, host))


def hard_decision(y):
    """z = (1 - sgn(y)) / 2 with sgn(0) = +1 (decoders.py:106-108): uint8."""
    torch = _torch()
    arr = y if isinstance(y, torch.Tensor) else np.asarray(y)
    dt = torch.float32 if arr.dtype in (np.float32, torch.float32) else torch.float64
    yt, host = _on_device(arr, dt)
    z = torch.empty(yt.shape, dtype=torch.uint8, device=yt.device)
    nat.check(nat.lib().fwbf_stage_hard_decision(4 if dt == torch.float32 else 8, yt.data_ptr(), yt.numel(),
                                                   z.data_ptr(), _stream(yt)), "hard_decision")
    return _out(z, host)


def syndrome(h, z):
    """z H^T over GF(2) (matrix.py:72-79), on the device; [N] or [B, N] uint8."""
    torch = _torch()
    zt, host = _on_device(z, torch.uint8)
    n = int(h.n_cols)
    if zt.shape[-1] != n or zt.dim() not in (1, 2):
        raise ValueError(f"expected a length-{n} vector")
    dc = _code(h, zt)
    batch = 1 if zt.dim() == 1 else int(zt.shape[0])
    s = torch.empty((dc.m,) if zt.dim() == 1 else (batch, dc.m), dtype=torch.uint8, device=zt.device)
    nat.check(nat.lib().fwbf_stage_syndrome(dc.handle, zt.data_ptr(), batch, s.data_ptr(), _stream(zt)),
              "syndrome")
    return _out(s, host)


def all_metrics(h, syndrome, edge_w, abs_y, alpha: float):
    """Eq.(1) metric of every bit for the given syndrome (decoders.py:148-153):
    the fp64 column sum in ascending check order, minus fl(alpha |y_n|)."""
    torch = _torch()
    st, host = _on_device(syndrome, torch.uint8)
    wt, _ = _on_device(edge_w, torch.float64)
    at, _ = _on_device(abs_y, torch.float64)
    dc = _code(h, st)
    batch = 1 if st.dim() == 1 else int(st.shape[0])
    if st.shape[-1] != dc.m or wt.shape[-1] != dc.n_edges or at.shape[-1] != dc.n:
        raise ValueError("syndrome / edge weight / |y| shapes do not match H")
    out = torch.empty(at.shape, dtype=torch.float64, device=st.device)
    nat.check(nat.lib().fwbf_stage_all_metrics(dc.handle, st.data_ptr(), wt.data_ptr(), at.data_ptr(),
                                                 float(alpha), batch, out.data_ptr(), _stream(st)), "all_metrics")
    return _out(out, host)


def block_argmax(values, p: int):
    """First maximum of each contiguous p-block, the tail padded with -inf
    (decoders.py:156-167); int64 [ceil(N/p)] (or [B, ceil(N/p)])."""
    torch = _torch()
    if p < 1:
        raise ValueError("block length p must be >= 1")
    vt, host = _on_device(values, torch.float64)
    n = int(vt.shape[-1])
    batch = 1 if vt.dim() == 1 else int(vt.shape[0])
    nb = -(-n // p)
    out = torch.empty((nb,) if vt.dim() == 1 else (batch, nb), dtype=torch.int64, device=vt.device)
    nat.check(nat.lib().fwbf_stage_block_argmax(vt.data_ptr(), batch, n, n, int(p), out.data_ptr(), _stream(vt)),
              "block_argmax")
    return _out(out, host)


def bit_metric(h, n: int, state, weights: WeightTable, y, alpha: float) -> float:
    """Metric of one bit straight from the definition (decoders.py:138-145):
    -alpha |y_n| first, then +-w per check of the column, ascending."""
    torch = _torch()
    st, _ = _on_device(state.syndrome, torch.uint8)
    m1, _ = _on_device(weights.min1, torch.float64)
    m2, _ = _on_device(weights.min2, torch.float64)
    am, _ = _on_device(weights.argmin_col, torch.int64)
    yt, _ = _on_device(y, torch.float64)
    dc = _code(h, st)
    if not 0 <= int(n) < dc.n:
        raise IndexError(f"bit index {n} out of range")
    cols = torch.tensor([int(n)], dtype=torch.int32, device=st.device)
    out = torch.empty(1, dtype=torch.float64, device=st.device)
    nat.check(nat.lib().fwbf_stage_bit_metric(dc.handle, cols.data_ptr(), 1, st.data_ptr(), m1.data_ptr(),
                                                m2.data_ptr(), am.data_ptr(), yt.data_ptr(), float(alpha),
                                                out.data_ptr(), _stream(st)), "bit_metric")
    return float(out.item())
