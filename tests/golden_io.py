"""Load the golden decode fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import glob
import json
import os
from dataclasses import dataclass
from typing import List

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class GoldenCase:
    name: str
    meta: dict
    y: np.ndarray
    z: np.ndarray            # uint8 [B, N]
    iterations: np.ndarray
    converged: np.ndarray
    stalled: np.ndarray
    flips_total: np.ndarray
    flip_logs: List[List[List[int]]]

    @property
    def decoder_kwargs(self) -> dict:
        m = self.meta
        return dict(alpha=m["alpha"], k_max=m["k_max"], lam=m["lam"], p=m["p"],
                    stall=m["stall"], mlp_threshold=m["mlp_threshold"],
                    weight_mode=m["weight_mode"])


def case_names() -> List[str]:
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if os.path.basename(p)[0] in "ABCDS")


def load_case(name: str) -> GoldenCase:
    d = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    meta = json.loads(str(d["meta"]))
    n = meta["n"]
    z = np.unpackbits(d["z"], axis=1)[:, :n]
    logs, pos, it = [], 0, 0
    iter_len = d["log_iter_len"]
    flat = d["log_flat"]
    for fl in d["log_frame_len"]:
        frame = []
        for _ in range(fl):
            k = int(iter_len[it])
            frame.append([int(v) for v in flat[pos:pos + k]])
            pos += k
            it += 1
        logs.append(frame)
    return GoldenCase(name, meta, d["y"], z, d["iterations"], d["converged"].astype(bool),
                      d["stalled"].astype(bool), d["flips_total"], logs)
