"""Named codes used by the fixtures and tests (built with the repo's constructors)."""

from __future__ import annotations

import functools

from paper_1206_3362_b200 import codes

# Information lengths K = N - rank_GF2(H), precomputed (test_host.py re-derives them).
_K = {"eg2": 7, "eg3": 37, "eg4": 175, "eg5": 781, "eg6": 3367,
      "gal504": 252, "qc4x32": 14339}


@functools.lru_cache(maxsize=None)
def build_code(name: str) -> codes.ParityCheckMatrix:
    if name.startswith("eg"):
        return codes.eg_ldpc(int(name[2:]))
    if name == "gal504":
        return codes.gallager_rc(504, 3, 6, seed=1)
    if name == "qc4x32":
        return codes.qc_ldpc(4, 32, 512, seed=2012)
    raise KeyError(name)


def code_k(name: str) -> int:
    return _K[name]


def code_rate(name: str) -> float:
    h = build_code(name)
    return _K[name] / h.n_cols
