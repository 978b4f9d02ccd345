"""The C ABI from a plain C program (examples/decode_host.c): no Python, no
CUDA headers in the client.  CPU: it compiles and links against the library.
GPU: its decode equals the oracle's, frame by frame."""
import os
import subprocess

import numpy as np
import pytest

from oracle import wbf_oracle as O
from paper_1206_3362_b200 import eg_ldpc
from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.codes import detect_structure

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_client(tmp_path):
    exe = str(tmp_path / "decode_host")
    libdir = os.path.dirname(nat.LIB_PATH)
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "examples", "decode_host.c"), "-L", libdir, "-lfwbf_b200",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True, capture_output=True)
    return exe


def test_c_client_builds(tmp_path):
    if not os.path.exists(nat.LIB_PATH):
        pytest.skip("library not built")
    assert os.path.exists(build_client(tmp_path))


@pytest.mark.gpu
def test_c_client_decodes_like_the_oracle(cuda_device, tmp_path):
    h = eg_ldpc(5)
    st = detect_structure(h)
    assert st.kind == "circulant"
    offsets = st.offsets
    n, B = h.n_cols, 24
    rng = np.random.default_rng(5)
    y = (1.0 + 0.55 * rng.standard_normal((B, n))).astype(np.float32)
    off_path, y_path = tmp_path / "off.bin", tmp_path / "y.bin"
    np.asarray(offsets, np.int32).tofile(off_path)
    y.tofile(y_path)
    exe = build_client(tmp_path)
    out = subprocess.run([exe, str(off_path), str(y_path), str(n), str(B), "31", "0.2", "100"],
                         check=True, capture_output=True, text=True).stdout.strip().splitlines()
    assert len(out) == B
    g = O.Graph.of(h)
    for f, line in enumerate(out):
        parts = line.split()
        r = O.decode(g, y[f], "fwbf", alpha=0.2, k_max=100, p=31)
        assert int(parts[0]) == r.iterations
        assert (int(parts[1]) & 1) == int(r.converged)
        words = np.array([int(w, 16) for w in parts[2:]], dtype=np.uint64)
        bits = ((words[:, None] >> np.arange(32, dtype=np.uint64)) & 1).astype(np.uint8).ravel()[:n]
        assert np.array_equal(bits, r.z)
