"""synth -- seeded synthetic inputs shared by the oracle and the CUDA path.

INPUT GENERATION ONLY: no step of the method's arithmetic lives here.  The
paper's corpora (Reuters-21578, a Wikipedia dump, PubMed abstracts;
PAPER.md:153,159,221,247-248) are not available, so seeded Zipf term/document
matrices with the shapes of BASELINE.json's configs stand in for them
(recipe in DESIGN.md section 3 and in synth/zipfgen.c).

* ``generate(cfg)``          -> numpy CSR(A) and CSR(A^T) (CPU, OpenMP C)
* ``generate_device(cfg)``   -> the same arrays built on the GPU (bitwise equal)
* ``CONFIGS``                -> the five BASELINE.json configs (BJ:7-11)
"""
from __future__ import annotations

import ctypes
import dataclasses
import functools
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_CPU_SO = os.path.join(HERE, "libzipfgen.so")
_CUDA_SO = os.path.join(HERE, "libzipfgen_cuda.so")
VTAB_BITS = 16


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config (BJ:7-11).  ``t=None`` means unlimited (Alg. 1)."""
    name: str
    n: int          # terms (rows of A)
    m: int          # documents (columns of A)
    d: int          # distinct terms per document
    s: float        # Zipf exponent of term ranks
    sigma: float    # lognormal sigma of values
    k: int          # rank (topics)
    t: int | None   # kept entries per topic column
    iters: int
    seed: int = 0

    @property
    def nnz(self) -> int:
        return self.m * self.d

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    # BJ:7  Tiny
    "tiny": Config("tiny", 2_000, 1_000, 50, 1.1, 1.0, 10, 50, 20),
    # BJ:8  Medium
    "medium": Config("medium", 50_000, 100_000, 100, 1.1, 1.0, 50, 500, 50),
    # BJ:9  Large
    "large": Config("large", 200_000, 1_000_000, 150, 1.05, 1.2, 100, 1_000, 50),
    # BJ:10 Box-scale
    "box": Config("box", 1_000_000, 8_000_000, 200, 1.05, 1.2, 200, 5_000, 30),
}
# BJ:11 sparsity sweep on the Medium matrix
SWEEP_T = (10, 100, 1_000, 10_000, None)


def build(verbose: bool = False) -> None:
    """Compile the CPU generator (gcc) and its CUDA twin (nvcc, sm_100a)."""
    src = os.path.join(HERE, "zipfgen.c")
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", src, "-o", _CPU_SO]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    srcu = os.path.join(HERE, "zipfgen_cuda.cu")
    cmdu = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
            "-Xcompiler", "-fPIC", srcu, "-o", _CUDA_SO]
    subprocess.run(cmdu, check=True, capture_output=not verbose)


def _needs_build(so: str, src: str) -> bool:
    return not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(HERE, src))


@functools.lru_cache(None)
def _cpu_lib():
    if _needs_build(_CPU_SO, "zipfgen.c"):
        build()
    lib = ctypes.CDLL(_CPU_SO)
    i64, i32, u64, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
    lib.zg_generate_at.argtypes = [i64, i64, i32, u64, p, p, p, p]
    lib.zg_generate_at.restype = ctypes.c_int
    lib.zg_transpose.argtypes = [i64, i64, p, p, p, p, p, p]
    lib.zg_transpose.restype = ctypes.c_int
    lib.zg_hash.argtypes = [u64, u64, u64, u64]
    lib.zg_hash.restype = u64
    return lib


@functools.lru_cache(None)
def _cuda_lib():
    if _needs_build(_CUDA_SO, "zipfgen_cuda.cu"):
        build()
    lib = ctypes.CDLL(_CUDA_SO)
    i64, i32, u64, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
    lib.zg_generate_at_cuda.argtypes = [i64, i64, i32, u64, p, p, p, p, p]
    lib.zg_generate_at_cuda.restype = ctypes.c_int
    return lib


@functools.lru_cache(None)
def zipf_cdf(n: int, s: float) -> np.ndarray:
    """cdf[r] = P(rank <= r) for P(rank = r) proportional to (r+1)^-s, r = 0..n-1."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    c = c / c[-1]
    c[-1] = 1.0
    return c


@functools.lru_cache(None)
def lognormal_vtab(sigma: float) -> np.ndarray:
    """65537 knots of the lognormal(0, sigma) quantile at p = (i+1)/65538."""
    from scipy.special import ndtri

    p = (np.arange((1 << VTAB_BITS) + 1, dtype=np.float64) + 1.0) / float((1 << VTAB_BITS) + 2)
    return np.exp(sigma * ndtri(p))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@functools.lru_cache(maxsize=4)
def generate(cfg: Config) -> dict:
    """CSR(A) (n x m, term rows) and CSR(A^T) (m x n, doc rows) as numpy arrays."""
    lib = _cpu_lib()
    n, m, d = cfg.n, cfg.m, cfg.d
    cdf = zipf_cdf(n, cfg.s)
    vtab = lognormal_vtab(cfg.sigma)
    at_col = np.empty(m * d, np.int32)
    at_val = np.empty(m * d, np.float32)
    rc = lib.zg_generate_at(n, m, d, cfg.seed, _ptr(cdf), _ptr(vtab), _ptr(at_col), _ptr(at_val))
    if rc != 0:
        raise ValueError(f"zg_generate_at failed for {cfg}")
    at_ptr = np.arange(m + 1, dtype=np.int64) * d
    a_ptr = np.empty(n + 1, np.int64)
    a_col = np.empty(m * d, np.int32)
    a_val = np.empty(m * d, np.float32)
    rc = lib.zg_transpose(n, m, _ptr(at_ptr), _ptr(at_col), _ptr(at_val), _ptr(a_ptr), _ptr(a_col), _ptr(a_val))
    if rc != 0:
        raise MemoryError("zg_transpose")
    out = dict(n=n, m=m, a_ptr=a_ptr, a_col=a_col, a_val=a_val, at_ptr=at_ptr, at_col=at_col, at_val=at_val)
    for v in out.values():
        if isinstance(v, np.ndarray):
            v.setflags(write=False)
    return out


def generate_device(cfg: Config, device="cuda", with_a: bool = True) -> dict:
    """The same matrices built in HBM (torch tensors).  A^T by the CUDA twin of
    zg_generate_at; A by a stable sort of the entries by term (torch plumbing)."""
    import torch

    lib = _cuda_lib()
    n, m, d = cfg.n, cfg.m, cfg.d
    dev = torch.device(device)
    cdf = torch.from_numpy(zipf_cdf(n, cfg.s)).to(dev)
    vtab = torch.from_numpy(lognormal_vtab(cfg.sigma)).to(dev)
    at_col = torch.empty(m * d, dtype=torch.int32, device=dev)
    at_val = torch.empty(m * d, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = lib.zg_generate_at_cuda(n, m, d, cfg.seed, cdf.data_ptr(), vtab.data_ptr(), at_col.data_ptr(),
                                 at_val.data_ptr(), stream)
    if rc != 0:
        raise RuntimeError(f"zg_generate_at_cuda failed ({rc})")
    at_ptr = torch.arange(m + 1, dtype=torch.int64, device=dev) * d
    out = dict(n=n, m=m, at_ptr=at_ptr, at_col=at_col, at_val=at_val)
    if with_a:
        order = torch.argsort(at_col, stable=True)
        a_col = (order // d).to(torch.int32)
        a_val = at_val[order]
        del order
        counts = torch.bincount(at_col.to(torch.int64), minlength=n)
        a_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        a_ptr[1:] = torch.cumsum(counts, 0)
        out.update(a_ptr=a_ptr, a_col=a_col, a_val=a_val)
    return out


def hash64(seed: int, stream: int, a: int, b: int) -> int:
    return int(_cpu_lib().zg_hash(seed, stream, a, b))
