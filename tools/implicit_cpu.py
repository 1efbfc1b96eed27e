"""ctypes wrapper of tools/implicit_cpu.c: CPU implicit dual-operator application (amortization
baseline, PAPER.md P:292-300 / P:2916-2919)."""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libimplicit_cpu.so")
_P = ctypes.c_void_p


def build_lib(force: bool = False) -> str:
    src = os.path.join(HERE, "implicit_cpu.c")
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared", "-o", LIB, src])
    return LIB


class _SD(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("Lp", _P), ("Li", _P), ("Lx", _P), ("iperm", _P),
                ("Bp", _P), ("Bi", _P), ("Bx", _P), ("lmap", _P)]


class ImplicitCPU:
    """Holds materialised per-subdomain arrays (L values included) and applies q = F lambda
    implicitly on the host cores."""

    def __init__(self, problem, threads: int = 0):
        self.lib = ctypes.CDLL(build_lib())
        self.lib.implicit_apply.restype = ctypes.c_int
        self.lib.implicit_apply.argtypes = [ctypes.c_int32, _P, _P, _P, ctypes.c_int64, _P, _P, _P, ctypes.c_int32,
                                            ctypes.c_int]
        self.keep = []
        subs = problem.subdomains
        self.sds = (_SD * len(subs))()
        yoff = [0]
        for i, sd in enumerate(subs):
            iperm = np.empty(sd.n, dtype=np.int32)
            iperm[sd.perm] = np.arange(sd.n, dtype=np.int32)
            arrs = [np.ascontiguousarray(sd.L_colptr, np.int64), np.ascontiguousarray(sd.L_rowidx, np.int32),
                    np.ascontiguousarray(sd.L_values, np.float64), iperm, np.ascontiguousarray(sd.Bt_colptr, np.int32),
                    np.ascontiguousarray(sd.Bt_rowidx, np.int32), np.ascontiguousarray(sd.Bt_values, np.float64),
                    np.ascontiguousarray(sd.lambda_map, np.int64)]
            self.keep.append(arrs)
            s = self.sds[i]
            s.n, s.m = sd.n, sd.m
            s.Lp, s.Li, s.Lx, s.iperm, s.Bp, s.Bi, s.Bx, s.lmap = [a.ctypes.data for a in arrs]
            yoff.append(yoff[-1] + sd.m)
        self.yoff = np.array(yoff[:-1], dtype=np.int64)
        self.ybuf = np.zeros(max(yoff[-1], 1))
        self.max_n = max(sd.n for sd in subs)
        self.threads = threads or len(os.sched_getaffinity(0))
        self.xbuf = np.zeros(self.threads * self.max_n + 1)
        self.n_lambda = problem.n_lambda
        self.nsub = len(subs)
        self.used_threads = self.threads

    def apply(self, lam: np.ndarray) -> np.ndarray:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        q = np.zeros(self.n_lambda)
        self.used_threads = self.lib.implicit_apply(self.nsub, self.sds, lam.ctypes.data, q.ctypes.data, self.n_lambda,
                                                    self.ybuf.ctypes.data, self.yoff.ctypes.data,
                                                    self.xbuf.ctypes.data, self.max_n, self.threads)
        return q

    def time(self, reps: int = 10, warmup: int = 2) -> float:
        """Median wall time (s) of one implicit apply over the whole batch."""
        lam = np.random.default_rng(0).standard_normal(self.n_lambda)
        for _ in range(warmup):
            self.apply(lam)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            self.apply(lam)
            ts.append(time.perf_counter() - t0)
        return float(np.median(ts))
