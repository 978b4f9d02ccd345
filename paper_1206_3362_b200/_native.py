"""ctypes binding of libfwbf_b200.so (the C ABI in include/fwbf_b200.h).

This is the same binding a maintainer would add to the reference package
(see INTEGRATION.md).  There is no fallback: if the library is missing or the
CUDA runtime cannot find a device, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# FWBF_LIB: development override (A/B builds of the same sources)
LIB_PATH = os.environ.get("FWBF_LIB") or os.path.join(_HERE, "libfwbf_b200.so")

FWBF_OK, FWBF_EINVAL, FWBF_ECUDA, FWBF_EUNSUPPORTED = 0, -1, -2, -3
ALG = {"fwbf": 0, "imwbf": 1, "mlp": 2}
WEIGHTS = {"imwbf": 0, "mwbf": 1}
STALL = {"flip-global-max": 0, "terminate": 1}
FLAG_CONVERGED, FLAG_STALLED, FLAG_ORDERED, FLAG_NONFINITE, FLAG_SPLIT32 = 1, 2, 4, 8, 16
NOISE_NUMPY_F64, NOISE_NUMPY_F32 = 0, 1
(CNT_FRAMES, CNT_BIT_ERRORS, CNT_WORD_ERRORS, CNT_ITER_SUM, CNT_FLIP_SUM, CNT_STALLS,
 CNT_CONVERGED, CNT_ORDERED_FRAMES, CNT_EDGE_VISITS, NCOUNTERS) = range(10)

EXPORTS = ("fwbf_abi_version", "fwbf_last_error", "fwbf_device_count", "fwbf_code_create",
           "fwbf_code_destroy", "fwbf_code_info", "fwbf_max_flips_per_iter", "fwbf_decode_f32",
           "fwbf_decode_f64", "fwbf_decode_awgn", "fwbf_decode_host_f32", "fwbf_metric_f32",
           "fwbf_metric_f64", "fwbf_filter_stats", "fwbf_stage_hard_decision", "fwbf_stage_syndrome",
           "fwbf_stage_weights", "fwbf_stage_edge_weights", "fwbf_stage_all_metrics", "fwbf_stage_block_argmax",
           "fwbf_stage_bit_metric", "fwbf_channel_awgn", "fwbf_last_kernel")


class CodeDesc(C.Structure):
    _fields_ = [("n_cols", C.c_int32), ("n_rows", C.c_int32),
                ("row_ptr", C.POINTER(C.c_int32)), ("row_idx", C.POINTER(C.c_int32)),
                ("circulant", C.c_int32), ("n_offsets", C.c_int32),
                ("offsets", C.POINTER(C.c_int32))]


class Params(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("weight_mode", C.c_int32), ("alpha", C.c_double),
                ("k_max", C.c_int32), ("lam", C.c_int32), ("block_len_p", C.c_int32),
                ("stall", C.c_int32), ("mlp_threshold", C.c_int32), ("force_ordered", C.c_int32)]


class Outputs(C.Structure):
    _fields_ = [("z_bits", C.c_void_p), ("z_ld", C.c_int64), ("iterations", C.c_void_p),
                ("flags", C.c_void_p), ("flips_total", C.c_void_p), ("bit_errors", C.c_void_p),
                ("fliplog", C.c_void_p), ("fliplog_counts", C.c_void_p),
                ("fliplog_stride", C.c_int64), ("counters", C.c_void_p),
                ("iter_hist", C.c_void_p), ("batch_word_err", C.c_void_p),
                ("batch_frames", C.c_int32), ("codeword_bits", C.c_void_p),
                ("y_out", C.c_void_p), ("y_out_ld", C.c_int64)]


class FwbfError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load the library once; raise if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1206_3362_b200.csrc.build`")
            L = C.CDLL(LIB_PATH)
            vp = C.c_void_p
            L.fwbf_abi_version.restype = C.c_int
            L.fwbf_last_error.restype = C.c_char_p
            L.fwbf_last_kernel.restype = C.c_char_p
            L.fwbf_device_count.restype = C.c_int
            L.fwbf_code_create.argtypes = [C.POINTER(CodeDesc), C.c_int, C.POINTER(vp)]
            L.fwbf_code_destroy.argtypes = [vp]
            L.fwbf_code_info.argtypes = [vp] + [C.POINTER(C.c_int32)] * 4
            L.fwbf_max_flips_per_iter.argtypes = [vp, C.POINTER(Params)]
            L.fwbf_max_flips_per_iter.restype = C.c_int64
            L.fwbf_decode_f32.argtypes = [vp, C.POINTER(Params), vp, C.c_int64, C.c_int64,
                                          C.POINTER(Outputs), vp]
            L.fwbf_decode_f64.argtypes = L.fwbf_decode_f32.argtypes
            L.fwbf_decode_awgn.argtypes = [vp, C.POINTER(Params), C.c_uint64, C.c_int64, C.c_int64,
                                           C.c_double, C.c_int32, C.POINTER(Outputs), vp]
            L.fwbf_decode_host_f32.argtypes = [vp, C.POINTER(Params), vp, C.c_int64, C.c_int64,
                                               vp, C.c_int64, vp, vp, vp, C.c_int64]
            L.fwbf_metric_f32.argtypes = [vp, C.POINTER(Params), vp, C.c_int64, C.c_int64, vp, C.c_int64,
                                          vp, vp]
            L.fwbf_metric_f64.argtypes = L.fwbf_metric_f32.argtypes
            L.fwbf_filter_stats.argtypes = [vp, C.POINTER(C.c_int64), C.c_int32]
            i64, i32, dbl = C.c_int64, C.c_int32, C.c_double
            L.fwbf_stage_hard_decision.argtypes = [i32, vp, i64, vp, vp]
            L.fwbf_stage_syndrome.argtypes = [vp, vp, i64, vp, vp]
            L.fwbf_stage_weights.argtypes = [vp, vp, i64, i64, vp, vp, vp, vp, vp]
            L.fwbf_stage_edge_weights.argtypes = [vp, vp, vp, vp, i64, vp, vp]
            L.fwbf_stage_all_metrics.argtypes = [vp, vp, vp, vp, dbl, i64, vp, vp]
            L.fwbf_stage_block_argmax.argtypes = [vp, i64, i64, i64, i32, vp, vp]
            L.fwbf_stage_bit_metric.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp, dbl, vp, vp]
            L.fwbf_channel_awgn.argtypes = [vp, C.c_uint64, i64, i64, dbl, vp, i32, vp, i64, vp]
            for f in EXPORTS:
                if f not in ("fwbf_abi_version", "fwbf_last_error", "fwbf_device_count",
                             "fwbf_max_flips_per_iter", "fwbf_last_kernel"):
                    getattr(L, f).restype = C.c_int
            if L.fwbf_abi_version() != 1:
                raise ImportError("libfwbf_b200.so ABI version mismatch")
            _lib = L
    return _lib


def last_kernel() -> str:
    """Kernel(s) this thread's last decode launched (diagnostic, fwbf_last_kernel)."""
    return lib().fwbf_last_kernel().decode()


def check(rc: int, what: str = "") -> None:
    if rc == FWBF_OK:
        return
    msg = lib().fwbf_last_error().decode(errors="replace")
    if rc == FWBF_EINVAL:
        raise ValueError(msg)
    raise FwbfError(f"{what}: {msg} (code {rc})")
