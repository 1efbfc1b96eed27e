"""CPU oracle for F_i = B~_i K_{i,reg}^{-1} B~_i^T — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may import
this package.  It shares no code with paper_2509_21037_b200/ (the CUDA path) and neither imports
the other.  The arithmetic lives in oracle/oracle.c (plain C, FP64; see its header for the steps
O1-O4 and the PAPER.md passages they follow); this file only marshals arrays through ctypes.

Parity status: every function here is pinned by tests/test_oracle_pins.py (brute-force dense
inverse, Schur-complement identity, 1D closed form, SPEC hand cases, invariants).
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Sequence

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_P = ctypes.c_void_p


def build_lib(force: bool = False) -> str:
    """Compile oracle/oracle.c into oracle/liboracle.so with gcc (plain C, -O2, no BLAS)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build_lib())
    lib.oracle_bandwidth.restype = ctypes.c_int32
    lib.oracle_bandwidth.argtypes = [ctypes.c_int32, _P, _P]
    lib.oracle_cholesky_band.restype = ctypes.c_int
    lib.oracle_cholesky_band.argtypes = [ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P]
    lib.oracle_forward.restype = None
    lib.oracle_forward.argtypes = [ctypes.c_int32, ctypes.c_int32, _P, _P]
    lib.oracle_backward.restype = None
    lib.oracle_backward.argtypes = [ctypes.c_int32, ctypes.c_int32, _P, _P]
    lib.oracle_dual_operator.restype = ctypes.c_int
    lib.oracle_dual_operator.argtypes = [ctypes.c_int32, _P, _P, _P, ctypes.c_int32, _P, _P, _P,
                                         ctypes.c_int32, _P, _P]
    return lib


def _csr(K):
    K = sp.csr_matrix(K)
    return (np.ascontiguousarray(K.indptr, dtype=np.int64), np.ascontiguousarray(K.indices, dtype=np.int32),
            np.ascontiguousarray(K.data, dtype=np.float64))


class OracleError(RuntimeError):
    pass


def cholesky(K) -> np.ndarray:
    """Dense lower L with K = L L^T (steps O1-O2), returned densely for tests."""
    rp, ci, v = _csr(K)
    n = K.shape[0]
    lib = _lib()
    b = lib.oracle_bandwidth(n, rp.ctypes.data, ci.ctypes.data)
    Lb = np.zeros(n * (b + 1))
    rc = lib.oracle_cholesky_band(n, b, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, Lb.ctypes.data)
    if rc != 0:
        raise OracleError(f"K not SPD at row {rc - 1}")
    L = np.zeros((n, n))
    Lb = Lb.reshape(n, b + 1)
    for i in range(n):
        for j in range(max(0, i - b), i + 1):
            L[i, j] = Lb[i, j - i + b]
    return L


def _band_from_dense(L: np.ndarray):
    n = L.shape[0]
    b = 0
    nz = np.nonzero(L)
    if len(nz[0]):
        b = int(np.max(np.abs(nz[0] - nz[1])))
    Lb = np.zeros((n, b + 1))
    for i in range(n):
        for j in range(max(0, i - b), i + 1):
            Lb[i, j - i + b] = L[i, j]
    return b, np.ascontiguousarray(Lb.ravel())


def forward(L: np.ndarray, x: np.ndarray) -> np.ndarray:
    """L^{-1} x with the oracle's forward substitution (step O3)."""
    b, Lb = _band_from_dense(np.asarray(L, dtype=np.float64))
    y = np.array(x, dtype=np.float64, copy=True)
    _lib().oracle_forward(len(y), b, Lb.ctypes.data, y.ctypes.data)
    return y


def backward(L: np.ndarray, x: np.ndarray) -> np.ndarray:
    """L^{-T} x with the oracle's backward substitution (step O3)."""
    b, Lb = _band_from_dense(np.asarray(L, dtype=np.float64))
    y = np.array(x, dtype=np.float64, copy=True)
    _lib().oracle_backward(len(y), b, Lb.ctypes.data, y.ctypes.data)
    return y


def dual_operator(K, Bt, cols: Optional[Sequence[int]] = None) -> np.ndarray:
    """F = B~ K^{-1} B~^T (m x m), or its columns `cols` (m x len(cols)), original multiplier order.

    K: SPD (n x n) sparse or dense, natural DOF order.  Bt: B~^T (n x m), sparse or dense."""
    rp, ci, v = _csr(K)
    n = K.shape[0]
    B = sp.csc_matrix(Bt)
    B.sort_indices()
    m = B.shape[1]
    bp = np.ascontiguousarray(B.indptr, dtype=np.int32)
    bi = np.ascontiguousarray(B.indices, dtype=np.int32)
    bv = np.ascontiguousarray(B.data, dtype=np.float64)
    if cols is None:
        nc, cptr, keep = m, None, None
    else:
        keep = np.ascontiguousarray(np.asarray(cols, dtype=np.int32))
        nc, cptr = len(keep), keep.ctypes.data
    F = np.zeros((nc, m))  # row c = column cols[c] of F (column-major m x nc)
    if m == 0 or nc == 0:
        return F.T.copy()
    rc = _lib().oracle_dual_operator(n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data, m, bp.ctypes.data,
                                     bi.ctypes.data, bv.ctypes.data, nc, cptr, F.ctypes.data)
    if rc != 0:
        raise OracleError("allocation failure" if rc < 0 else f"K not SPD at row {rc - 1}")
    return F.T.copy()


def subdomain_F(sd, cols: Optional[Sequence[int]] = None) -> np.ndarray:
    """Oracle F for one synth.Subdomain (uses only K_reg and B~^T, never L or perm)."""
    return dual_operator(sd.K_reg, sd.Bt_sparse(), cols)


def batch_F(subdomains, threads: int = 0, cols=None):
    """Oracle over many subdomains, one subdomain per host thread (ctypes releases the GIL)."""
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda sd: subdomain_F(sd, cols), subdomains))
