"""The C-ABI library: builds, loads and exports every symbol include/esnmf.h
declares (CPU only -- no compute calls), plus the host-only helpers."""
import os
import re

import numpy as np
import pytest

import paper_1510_05237_b200 as pk
from paper_1510_05237_b200 import esnmf as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "esnmf.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(esnmf_[A-Za-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for s in ("esnmf_create", "esnmf_iterate", "esnmf_residual", "esnmf_error", "esnmf_get_U", "esnmf_get_V",
              "esnmf_destroy"):
        assert s in syms


def test_library_loads_and_exports_every_declared_symbol():
    L = pk.lib()
    syms = header_symbols()
    assert syms
    for s in syms:
        assert hasattr(L, s), s
        assert s in B.SIGNATURES, f"binding lacks {s}"
    assert "sm_100a" in pk.esnmf_version()


def test_library_is_built_for_sm100a():
    import subprocess

    so = B._build.SO
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_strerror_and_options_defaults():
    L = pk.lib()
    assert L.esnmf_strerror(0) == b"ok"
    assert L.esnmf_strerror(8) == b"buffer too small"
    o = pk.esnmf_options_init()
    assert o.seed == 0 and o.ridge_scale == 1e-10 and o.world == 1 and o.rank == 0 and o.device == -1
    assert not o.stream and not o.at_row_ptr and not o.U0


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the header structs have the C compiler's size and offsets."""
    import ctypes
    import subprocess

    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "esnmf.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(esnmf_options), sizeof(esnmf_record),"
        " sizeof(esnmf_info), sizeof(esnmf_comm), offsetof(esnmf_options, inputs_on_device),"
        " offsetof(esnmf_record, active_v), offsetof(esnmf_info, normA2), sizeof(esnmf_cost),"
        " offsetof(esnmf_cost, v_tail_gather)); return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(B.esnmf_options), ctypes.sizeof(B.esnmf_record), ctypes.sizeof(B.esnmf_info),
            ctypes.sizeof(B.esnmf_comm), B.esnmf_options.inputs_on_device.offset, B.esnmf_record.active_v.offset,
            B.esnmf_info.normA2.offset, ctypes.sizeof(B.esnmf_cost), B.esnmf_cost.v_tail_gather.offset]
    assert got == want


def test_partition_rows_balances_nnz():
    rng = np.random.default_rng(0)
    lens = (rng.zipf(1.3, 5000) % 2000).astype(np.int64)
    ptr = np.concatenate([[0], np.cumsum(lens)])
    for world in (1, 2, 3, 8):
        b = pk.esnmf_partition_rows(ptr, world)
        assert b[0] == 0 and b[-1] == len(lens) and np.all(np.diff(b) >= 0)
        cost = np.array([ptr[b[p + 1]] - ptr[b[p]] + (b[p + 1] - b[p]) for p in range(world)])
        assert cost.max() <= (ptr[-1] + len(lens)) / world + lens.max() + 1
    with pytest.raises(B.ESNMFError):
        pk.esnmf_partition_rows(ptr, 0)
