"""Thin Python binding of the C ABI in include/sc_b200.h (argument marshalling only).

Every step of the hot path runs in libsc_b200.so (sm_100a kernels); this module only converts numpy
arrays / torch tensors into the pointers and sizes the ABI takes.  There is no CPU fallback: if the
library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SC_B200_LIB: alternative in-tree build for A/B measurements (tools/); default the in-tree library
LIB_PATH = os.environ.get("SC_B200_LIB") or os.path.join(HERE, "libsc_b200.so")

SC_OK, SC_ERR_INVALID_ARG, SC_ERR_PATTERN, SC_ERR_ZERO_PIVOT, SC_ERR_OOM, SC_ERR_CUDA, SC_ERR_STATE = range(7)
SKIP_NONE, SKIP_ENVELOPE, SKIP_EXACT = 0, 1, 2
STRIP_AUTO, STRIP_SHARED, STRIP_GLOBAL = 0, 1, 2
TRSM_AUTO, TRSM_CTA, TRSM_WARP = 0, 1, 2
_STATUS = {0: "SC_OK", 1: "SC_ERR_INVALID_ARG", 2: "SC_ERR_PATTERN", 3: "SC_ERR_ZERO_PIVOT", 4: "SC_ERR_OOM",
           5: "SC_ERR_CUDA", 6: "SC_ERR_STATE"}

_P = ctypes.c_void_p


class ScError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class SubdomainDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("L_colptr", _P), ("L_rowidx", _P), ("perm", _P),
                ("Bt_colptr", _P), ("Bt_rowidx", _P), ("Bt_values", _P), ("lambda_map", _P)]


class Options(ctypes.Structure):
    _fields_ = [("precision", ctypes.c_int32), ("skip", ctypes.c_int32), ("tile_cols", ctypes.c_int32),
                ("panel_cols", ctypes.c_int32), ("n_lambda_global", ctypes.c_int64), ("device", ctypes.c_int32),
                ("x_strip", ctypes.c_int32), ("trsm_kernel", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5)]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in ("nsub", "n_classes", "tile_cols", "panel_cols")] + \
               [(k, ctypes.c_int64) for k in ("sum_n", "sum_m", "max_m", "sum_nnz_L", "trsm_tasks", "trsm_steps",
                                              "syrk_tasks", "syrk_segments")] + \
               [(k, ctypes.c_double) for k in ("flops_trsm_useful", "flops_syrk_useful", "flops_trsm_envelope",
                                               "flops_syrk_envelope", "flops_trsm_dense", "flops_syrk_dense",
                                               "flops_trsm_sparse_orig", "flops_trsm_executed",
                                               "flops_syrk_executed", "bytes_L_values", "bytes_F_lower", "bytes_X",
                                               "device_bytes", "bytes_apply", "bytes_panels")] + \
               [("panels", ctypes.c_int64), ("group_cols", ctypes.c_int32), ("x_strip", ctypes.c_int32),
                ("trsm_tasks_2cta", ctypes.c_int64), ("trsm_kernel", ctypes.c_int32), ("pad0", ctypes.c_int32),
                ("bytes_X_reach", ctypes.c_double), ("flops_factor_useful", ctypes.c_double),
                ("flops_factor_executed", ctypes.c_double), ("bytes_K_values", ctypes.c_double),
                ("factor_tasks", ctypes.c_int64), ("factor_panels", ctypes.c_int64),
                ("factor_max_level", ctypes.c_int32), ("pad1", ctypes.c_int32), ("bytes_factor_W", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class KPattern(ctypes.Structure):
    _fields_ = [("K_colptr", _P), ("K_rowidx", _P)]


class Coarse(ctypes.Structure):
    _fields_ = [("nc", ctypes.c_int32), ("k", _P), ("off", _P), ("Rt", _P), ("GtG_inv", _P)]


class PcpgOpts(ctypes.Structure):
    _fields_ = [("rtol", ctypes.c_double), ("max_it", ctypes.c_int32), ("alpha", _P)]


class PcpgResult(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("rel_residual", ctypes.c_double), ("history", _P),
                ("history_len", ctypes.c_int32)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)


class _DeviceBuf:
    """Zero-copy view of a device buffer handed to the all-reduce callback (CUDA array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


_lib = None

EXPORTS = ["sc_pcpg", "sc_options_default", "sc_plan_create", "sc_assemble_batch", "sc_assemble_batch_host", "sc_apply",
           "sc_check", "sc_get_F", "sc_get_X", "sc_plan_strip_rows", "sc_plan_stats", "sc_plan_subdomain_costs",
           "sc_set_timing_events", "sc_launches_per_assemble",
           "sc_launches_per_apply", "sc_plan_destroy", "sc_last_error", "sc_prepare_factor", "sc_apply_implicit",
           "sc_launches_per_apply_implicit", "sc_factor_attach", "sc_factorize_batch", "sc_factorize_assemble_host",
           "sc_get_F_device"]


def lib():
    """Load libsc_b200.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    L.sc_options_default.argtypes = [ctypes.POINTER(Options)]
    L.sc_options_default.restype = None
    L.sc_plan_create.argtypes = [ctypes.POINTER(SubdomainDesc), ctypes.c_int32, ctypes.POINTER(Options), ctypes.POINTER(_P)]
    L.sc_assemble_batch.argtypes = [_P, ctypes.POINTER(_P), _P]
    L.sc_assemble_batch_host.argtypes = [_P, ctypes.POINTER(_P), _P]
    L.sc_apply.argtypes = [_P, _P, _P, _P]
    L.sc_check.argtypes = [_P]
    L.sc_prepare_factor.argtypes = [_P, ctypes.POINTER(_P), _P]
    L.sc_apply_implicit.argtypes = [_P, _P, _P, _P]
    L.sc_launches_per_apply_implicit.argtypes = [_P]
    L.sc_launches_per_apply_implicit.restype = ctypes.c_int32
    L.sc_get_F.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int64]
    L.sc_get_X.argtypes = [_P, ctypes.c_int32, _P, _P]
    L.sc_get_F_device.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int64, _P]
    L.sc_plan_strip_rows.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, _P, _P]
    L.sc_plan_stats.argtypes = [_P, ctypes.POINTER(Stats)]
    L.sc_set_timing_events.argtypes = [_P, _P, ctypes.c_int32]
    L.sc_plan_subdomain_costs.argtypes = [_P, _P]
    L.sc_launches_per_assemble.argtypes = [_P]
    L.sc_launches_per_assemble.restype = ctypes.c_int32
    L.sc_launches_per_apply.argtypes = [_P]
    L.sc_launches_per_apply.restype = ctypes.c_int32
    L.sc_plan_destroy.argtypes = [_P]
    L.sc_plan_destroy.restype = None
    L.sc_pcpg.argtypes = [_P, _P, _P, _P, ctypes.POINTER(Coarse), ctypes.POINTER(PcpgOpts), ALLREDUCE_FN, _P,
                          ctypes.POINTER(PcpgResult), _P]
    L.sc_pcpg.restype = ctypes.c_int
    L.sc_factor_attach.argtypes = [_P, ctypes.POINTER(KPattern), ctypes.c_int32]
    L.sc_factorize_batch.argtypes = [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), _P]
    L.sc_factorize_assemble_host.argtypes = [_P, ctypes.POINTER(_P), _P]
    L.sc_last_error.argtypes = []
    L.sc_last_error.restype = ctypes.c_char_p
    for f in ("sc_plan_create", "sc_assemble_batch", "sc_assemble_batch_host", "sc_apply", "sc_check", "sc_get_F",
              "sc_prepare_factor", "sc_apply_implicit", "sc_factor_attach", "sc_factorize_batch",
              "sc_factorize_assemble_host", "sc_get_F_device",
              "sc_get_X", "sc_plan_strip_rows", "sc_plan_stats", "sc_set_timing_events", "sc_plan_subdomain_costs"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(status: int):
    if status != SC_OK:
        raise ScError(status, lib().sc_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class SCPlan:
    """sc_plan_create + the three stages.  `subdomains`: objects with n, m, L_colptr, L_rowidx, perm,
    Bt_colptr, Bt_rowidx, Bt_values, lambda_map (numpy arrays, e.g. synth.Subdomain)."""

    def __init__(self, subdomains: Sequence, *, n_lambda: int = 0, skip: int = SKIP_EXACT, tile_cols: int = 0,
                 panel_cols: int = 0, device: int = 0, x_strip: int = STRIP_AUTO,
                 trsm_kernel: int = TRSM_AUTO, precision: int = 64):
        L = lib()
        keep: List[np.ndarray] = []

        def arr(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        descs = (SubdomainDesc * max(len(subdomains), 1))()
        self.n = []
        self.m = []
        self.nnz = []
        for i, sd in enumerate(subdomains):
            d = descs[i]
            d.n, d.m = int(sd.n), int(sd.m)
            d.L_colptr = _ptr(arr(sd.L_colptr, np.int64))
            d.L_rowidx = _ptr(arr(sd.L_rowidx, np.int32))
            d.perm = _ptr(arr(getattr(sd, "perm", None), np.int32))
            d.Bt_colptr = _ptr(arr(sd.Bt_colptr, np.int32))
            d.Bt_rowidx = _ptr(arr(sd.Bt_rowidx, np.int32))
            d.Bt_values = _ptr(arr(sd.Bt_values, np.float64))
            d.lambda_map = _ptr(arr(getattr(sd, "lambda_map", None), np.int64))
            self.n.append(d.n)
            self.m.append(d.m)
            self.nnz.append(int(sd.L_colptr[-1]))
        opt = Options()
        L.sc_options_default(ctypes.byref(opt))
        opt.skip, opt.tile_cols, opt.panel_cols, opt.x_strip = skip, tile_cols, panel_cols, x_strip
        opt.trsm_kernel = trsm_kernel
        opt.precision = int(precision)
        self.precision = int(precision)
        opt.n_lambda_global, opt.device = int(n_lambda), int(device)
        self.device = device
        self.n_lambda = int(n_lambda)
        h = _P()
        _check(L.sc_plan_create(descs, len(subdomains), ctypes.byref(opt), ctypes.byref(h)))
        self._h = h
        self.nsub = len(subdomains)

    # -- preprocessing
    def pointer_array(self, L_values: Sequence):
        """The C pointer array (void*[nsub]) of per-subdomain value buffers, for reuse across calls:
        assemble / assemble_host / prepare_factor accept it in place of the list (no per-call
        marshalling of nsub Python objects)."""
        return self._value_ptrs(L_values)

    def _value_ptrs(self, L_values: Sequence):
        """Pointer array of the per-subdomain L values; tensors must have the plan's element type
        (float64, or float32 for precision 32).  A pointer array from pointer_array() passes through."""
        if isinstance(L_values, ctypes.Array):
            if len(L_values) < max(self.nsub, 1):
                raise ValueError("pointer array shorter than the number of subdomains")
            return L_values
        ptrs = (_P * max(self.nsub, 1))()
        want = 8 if self.precision == 64 else 4
        for i, t in enumerate(L_values):
            if isinstance(t, int):
                ptrs[i] = t
                continue
            esz = t.element_size() if hasattr(t, "element_size") else t.itemsize
            if esz != want:
                raise TypeError(f"L_values[{i}]: {want}-byte elements expected for precision {self.precision}")
            ptrs[i] = t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
        return ptrs

    def assemble(self, L_values: Sequence, stream=None):
        """L_values: per subdomain a CUDA tensor (float64, or float32 for precision 32) or a raw device
        pointer (int) of nnz(L) values."""
        _check(lib().sc_assemble_batch(self._h, self._value_ptrs(L_values), _stream_handle(stream)))

    def assemble_host(self, L_values: Sequence[np.ndarray], stream=None):
        """L values in host memory (pinned torch tensors or numpy arrays); copied H2D inside the call."""
        _check(lib().sc_assemble_batch_host(self._h, self._value_ptrs(L_values), _stream_handle(stream)))

    # -- device numeric factorization
    def factor_attach(self, K_patterns: Sequence):
        """K_patterns: per subdomain (K_colptr, K_rowidx) of the LOWER triangle of K_reg in the original
        DOF numbering (e.g. scipy tril(K).tocsc() indptr / indices)."""
        keep = []
        pats = (KPattern * max(self.nsub, 1))()
        for i, (cp, ri) in enumerate(K_patterns):
            a = np.ascontiguousarray(cp, dtype=np.int64)
            b = np.ascontiguousarray(ri, dtype=np.int32)
            keep += [a, b]
            pats[i].K_colptr, pats[i].K_rowidx = a.ctypes.data, b.ctypes.data
        _check(lib().sc_factor_attach(self._h, pats, self.nsub))
        self.nnzK = [int(cp[-1]) for cp, _ in K_patterns]

    def factorize(self, K_values: Sequence, L_out: Sequence, stream=None):
        """K_values: per subdomain a CUDA float64 tensor (or device pointer) of nnz(K) values; L_out:
        CUDA tensors (float64, or float32 for precision 32) of nnz(L) values, written."""
        kp = (_P * max(self.nsub, 1))()
        for i, t in enumerate(K_values):
            kp[i] = t if isinstance(t, int) else t.data_ptr()
        _check(lib().sc_factorize_batch(self._h, kp, self._value_ptrs(L_out), _stream_handle(stream)))

    def factorize_assemble_host(self, K_values: Sequence, stream=None):
        """K values in host memory (pinned float64 tensors or numpy arrays): H2D copy of K, device
        factorization, assembly -- all inside the call."""
        if isinstance(K_values, ctypes.Array):  # from pointer_array()
            kp = K_values
        else:
            kp = (_P * max(self.nsub, 1))()
            for i, t in enumerate(K_values):
                kp[i] = t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data
        _check(lib().sc_factorize_assemble_host(self._h, kp, _stream_handle(stream)))

    # -- solution
    def prepare_factor(self, L_values: Sequence, stream=None):
        """Stage the factor panels only (no F): what apply_implicit needs."""
        _check(lib().sc_prepare_factor(self._h, self._value_ptrs(L_values), _stream_handle(stream)))

    def apply_implicit(self, lam, q, stream=None):
        """q <- sum_i scatter(B~_i K_i^{-1} B~_i^T gather(lam)) without F (two substitutions per subdomain)."""
        _check(lib().sc_apply_implicit(self._h, lam.data_ptr(), q.data_ptr(), _stream_handle(stream)))

    def apply(self, lam, q, stream=None):
        """q <- sum_i scatter(F_i gather(lam)) over this plan's subdomains (device tensors, float64)."""
        _check(lib().sc_apply(self._h, lam.data_ptr(), q.data_ptr(), _stream_handle(stream)))

    def apply_global(self, lam, q, group=None, stream=None):
        """sc_apply then all-reduce(sum) of q over the ranks of `group` (NCCL over NVLink)."""
        import torch.distributed as dist
        self.apply(lam, q, stream)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(q, op=dist.ReduceOp.SUM, group=group)

    def pcpg(self, d, lam, *, e=None, coarse=None, rtol: float = 1e-10, max_it: int = 1000, alpha=None,
             group=None, history: int = 0, stream=None):
        """PCPG on the FETI dual problem (sc_pcpg): d, lam device float64 tensors (n_lambda); e host
        array (nc) of R^T f; coarse = dict(nc, k (per subdomain of this plan), off, Rt (device tensors
        B~_i R_i, m_i x k_i, column-major, original multiplier order), GtG_inv (device nc x nc));
        alpha: optional device tensor (nc) receiving alpha.  For N > 1 ranks the partial F p, G^T x
        and G y are summed with torch.distributed.all_reduce (NCCL).  Returns (iterations, final
        relative residual, residual history)."""
        import torch
        import torch.distributed as dist
        keep = []
        cs = None
        if coarse is not None and int(coarse["nc"]) > 0:
            k = np.ascontiguousarray(coarse["k"], dtype=np.int32)
            off = np.ascontiguousarray(coarse["off"], dtype=np.int64)
            rt = (_P * max(self.nsub, 1))(*[t.data_ptr() for t in coarse["Rt"]])
            keep += [k, off, rt, coarse["Rt"], coarse["GtG_inv"]]
            cs = Coarse(int(coarse["nc"]), k.ctypes.data, off.ctypes.data, ctypes.cast(rt, _P),
                        coarse["GtG_inv"].data_ptr())
        e_arr = None
        if e is not None:
            e_arr = np.ascontiguousarray(e, dtype=np.float64)
            keep.append(e_arr)
        opts = PcpgOpts(float(rtol), int(max_it), None if alpha is None else alpha.data_ptr())
        hist = np.zeros(max(history, 1))
        res = PcpgResult(0, 0.0, hist.ctypes.data if history else None, int(history))
        cb = ALLREDUCE_FN()
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            def _allreduce(ptr, n, ctx):
                dist.all_reduce(torch.as_tensor(_DeviceBuf(ptr, n), device="cuda"), group=group)
            cb = ALLREDUCE_FN(_allreduce)
        _check(lib().sc_pcpg(self._h, d.data_ptr(), None if e_arr is None else e_arr.ctypes.data, lam.data_ptr(),
                             ctypes.byref(cs) if cs is not None else None, ctypes.byref(opts), cb, None,
                             ctypes.byref(res), _stream_handle(stream)))
        return res.iterations, res.rel_residual, hist[:min(history, res.iterations + 1)] if history else None

    # -- queries
    def check(self):
        _check(lib().sc_check(self._h))

    def get_F(self, i: int) -> np.ndarray:
        m = self.m[i]
        F = np.zeros((m, m), dtype=np.float64, order="F")
        _check(lib().sc_get_F(self._h, i, F.ctypes.data, m))
        return np.asfortranarray(F)

    def get_F_device(self, i: int, out=None, stream=None):
        """F_i (full symmetric, original multiplier order) into a CUDA float64 tensor (m x m, column-major:
        out[b, a] = F(a, b), i.e. the transpose view of a row-major tensor; F is symmetric anyway)."""
        import torch
        m = self.m[i]
        if out is None:
            out = torch.empty((m, m), dtype=torch.float64, device=f"cuda:{self.device}")
        _check(lib().sc_get_F_device(self._h, i, out.data_ptr(), m, _stream_handle(stream)))
        return out

    def get_X(self, i: int):
        n, m = self.n[i], self.m[i]
        X = np.zeros((n, m), dtype=np.float64, order="F")
        sigma = np.zeros(max(m, 1), dtype=np.int32)
        _check(lib().sc_get_X(self._h, i, X.ctypes.data, sigma.ctypes.data))
        return X, sigma[:m]

    def sigma(self, i: int) -> np.ndarray:
        sigma = np.zeros(max(self.m[i], 1), dtype=np.int32)
        _check(lib().sc_get_X(self._h, i, None, sigma.ctypes.data))
        return sigma[:self.m[i]]

    def strip_rows(self, i: int, a: int) -> np.ndarray:
        rows = np.zeros(max(self.n[i], 1), dtype=np.int32)
        k = ctypes.c_int32(0)
        _check(lib().sc_plan_strip_rows(self._h, i, a, rows.ctypes.data, ctypes.addressof(k)))
        return rows[:k.value]

    def subdomain_costs(self) -> np.ndarray:
        c = np.zeros(max(self.nsub, 1))
        _check(lib().sc_plan_subdomain_costs(self._h, c.ctypes.data))
        return c[:self.nsub]

    def stats(self) -> dict:
        s = Stats()
        _check(lib().sc_plan_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def set_timing_events(self, events=None):
        """4 torch.cuda.Event objects (already recorded once, so they exist) recorded before prep,
        after prep, after the TRSM and after the SYRK of each following assemble; None disables."""
        if not events:
            _check(lib().sc_set_timing_events(self._h, None, 0))
            return
        arr = (_P * 4)(*[e.cuda_event for e in events])
        self._tev_keep = (events, arr)
        _check(lib().sc_set_timing_events(self._h, arr, 4))

    @property
    def launches_per_assemble(self) -> int:
        return lib().sc_launches_per_assemble(self._h)

    @property
    def launches_per_apply(self) -> int:
        return lib().sc_launches_per_apply(self._h)

    def destroy(self):
        if getattr(self, "_h", None):
            lib().sc_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
