"""C-ABI library: builds, loads, exports every declared symbol; fails loudly without a GPU."""

import os
import re

import numpy as np
import pytest

from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.csrc import build as B

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(REPO, "include", "fwbf_b200.h")).read()
    return sorted(set(re.findall(r"\b(fwbf_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_all_declared_symbols():
    B.build()
    L = nat.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(nat.EXPORTS)
    assert L.fwbf_abi_version() == 1


def test_ctypes_struct_layout_matches_header(tmp_path):
    """Compile a probe against include/fwbf_b200.h and compare every offset."""
    import ctypes as C
    import subprocess
    structs = {"fwbf_code_desc": nat.CodeDesc, "fwbf_params": nat.Params, "fwbf_outputs": nat.Outputs}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "fwbf_b200.h"', "int main(void){"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l}
    for cname, py in structs.items():
        assert got[(cname, "size")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


@pytest.mark.skipif(nat.lib().fwbf_device_count() > 0, reason="GPU present")
def test_no_silent_cpu_fallback():
    from paper_1206_3362_b200 import eg_ldpc
    from paper_1206_3362_b200.decoders import DeviceCode
    with pytest.raises(nat.FwbfError):
        DeviceCode(eg_ldpc(2))
