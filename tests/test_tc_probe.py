"""tcgen05 building blocks (csrc/tc.cuh) against numpy: layout, descriptors,
TMEM round trip and the 3xTF32 split accuracy the V-side head GEMM relies on."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tc_probe.cu")
SO = os.path.join(HERE, "libtc_probe.so")


def build():
    if not os.path.exists(SO) or os.path.getmtime(SO) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "..", "paper_1510_05237_b200", "csrc", "tc.cuh"))):
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                        "-Xcompiler", "-fPIC", SRC, "-o", SO], check=True)
    lib = ctypes.CDLL(SO)
    lib.tc_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 3
    return lib


def test_tc_probe_builds():
    build()


@pytest.mark.gpu
@pytest.mark.parametrize("K,N", [(8, 16), (64, 112), (32, 64), (64, 208)])
def test_tcgen05_tf32_gemm(K, N):
    lib = build()
    rng = np.random.default_rng(K * 1000 + N)
    A = rng.lognormal(0, 1, (128, K)).astype(np.float32)
    B = rng.normal(0, 1, (N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    scale = np.abs(ref).max(axis=0)
    for split, tol in ((0, 5e-3), (1, 2e-6)):
        D = np.zeros((128, N), np.float32)
        rc = lib.tc_probe(A.ctypes.data, B.ctypes.data, D.ctypes.data, K, N, split)
        assert rc == 0
        err = (np.abs(D - ref) / scale).max()
        assert err < tol, (split, err)
