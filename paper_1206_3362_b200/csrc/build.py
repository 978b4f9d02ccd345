"""Build libfwbf_b200.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

    python -m paper_1206_3362_b200.csrc.build        # or build() from __graft_entry__

The library is plain C-ABI (include/fwbf_b200.h); the CUDA runtime is linked
statically so the .so only needs the driver at run time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
REPO = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libfwbf_b200.so")
SOURCES = ["fwbf_decode.cu", "fwbf_circ.cu", "fwbf_explicit.cu", "fwbf_qc.cu", "fwbf_noise.cu", "fwbf_stage.cu", "fwbf_api.cu"]
HEADERS = ["fwbf_internal.h", "fwbf_noise.cuh", "fwbf_device.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, s) for s in SOURCES + HEADERS] + [
        os.path.join(REPO, "include", "fwbf_b200.h"), os.path.abspath(__file__)]
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB) -> str:
    if out == LIB and not force and not _stale():
        return LIB
    srcs = [os.path.join(HERE, s) for s in SOURCES if os.path.exists(os.path.join(HERE, s))]
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-cudart", "static", "-fmad=false", "--expt-relaxed-constexpr",
           "-static-global-template-stub=false",
           "-I", os.path.join(REPO, "include"), "-I", HERE,
           "-Xptxas", "-v" if verbose else "-O3",
           *os.environ.get("FWBF_EXTRA_NVCC", "").split(),
           "-o", out + ".tmp", *srcs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libfwbf_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    outs = [a[len("--out="):] for a in sys.argv if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=os.path.abspath(outs[0]) if outs else LIB))
