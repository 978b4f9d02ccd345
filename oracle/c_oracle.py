"""ctypes loader for oracle/libwbf_oracle.so -- TEST INFRASTRUCTURE ONLY.

A C restatement of the same reference algorithm as wbf_oracle.py (see the
header of wbf_oracle.c), used as a fast independent checker for large batches.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libwbf_oracle.so")
ALG = {"fwbf": 0, "imwbf": 1, "mlp": 2}


class _Code(C.Structure):
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("row_ptr", C.c_void_p), ("row_idx", C.c_void_p),
                ("col_ptr", C.c_void_p), ("col_idx", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("algorithm", C.c_int), ("weight_mode", C.c_int), ("alpha", C.c_double),
                ("k_max", C.c_int), ("lam", C.c_int), ("p", C.c_int), ("stall", C.c_int),
                ("mlp_threshold", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        L = C.CDLL(LIB)
        L.orc_decode_batch.argtypes = [C.POINTER(_Code), C.POINTER(_Params), C.c_void_p, C.c_int,
                                       C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        L.orc_decode.argtypes = [C.POINTER(_Code), C.POINTER(_Params), C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_decode.restype = C.c_int
        _lib = L
    return _lib


class COracle:
    def __init__(self, h):
        rows = [np.asarray(r, dtype=np.int64) for r in h.row_adj]
        n, m = int(h.n_cols), len(rows)
        self.n, self.m = n, m
        self.row_ptr = np.zeros(m + 1, np.int32)
        np.cumsum([r.size for r in rows], out=self.row_ptr[1:])
        self.row_idx = np.concatenate(rows).astype(np.int32)
        er = np.repeat(np.arange(m), np.diff(self.row_ptr))
        order = np.argsort(self.row_idx, kind="stable")
        self.col_idx = er[order].astype(np.int32)
        self.col_ptr = np.zeros(n + 1, np.int32)
        np.cumsum(np.bincount(self.row_idx, minlength=n), out=self.col_ptr[1:])
        self.code = _Code(n, m, self.row_ptr.ctypes.data, self.row_idx.ctypes.data,
                          self.col_ptr.ctypes.data, self.col_idx.ctypes.data)

    def params(self, algorithm="fwbf", alpha=0.2, k_max=10, lam=1, p=1, stall="flip-global-max",
               mlp_threshold=True, weight_mode="imwbf"):
        return _Params(ALG[algorithm], 0 if weight_mode == "imwbf" else 1, float(alpha), int(k_max),
                       int(lam), int(p or 0), 0 if stall == "flip-global-max" else 1,
                       1 if mlp_threshold else 0)

    def decode_batch(self, y, threads=None, **kw):
        """(z uint8 [B,N], iterations, flags, flips_total) for y [B,N] float32/float64."""
        y = np.ascontiguousarray(y)
        if y.dtype not in (np.float32, np.float64):
            y = y.astype(np.float64)
        B = y.shape[0]
        prm = self.params(**kw)
        z = np.zeros((B, self.n), np.uint8)
        its = np.zeros(B, np.int32)
        fl = np.zeros(B, np.int32)
        ft = np.zeros(B, np.int32)
        L = lib()
        threads = threads or min(32, os.cpu_count() or 1)
        chunks = [(s, min(B, s + max(1, B // threads))) for s in range(0, B, max(1, B // threads))]

        def run(c):
            s, e = c
            L.orc_decode_batch(C.byref(self.code), C.byref(prm), y[s:e].ctypes.data,
                               1 if y.dtype == np.float64 else 0, e - s, self.n,
                               z[s:e].ctypes.data, its[s:e].ctypes.data, fl[s:e].ctypes.data,
                               ft[s:e].ctypes.data)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, chunks))
        return z, its, fl, ft
