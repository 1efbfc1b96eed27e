"""Structured Q1 FETI problems: meshes, decomposition, gluing, regularisation, ordering, factor.

Input generation only (see synth/__init__.py).  Paper context: heat transfer on a unit square/cube,
"uniformly discretized" and decomposed into subdomains (§4); block FETI system
with signed-Boolean gluing B (eq. fetisystemblocked); regularised K_{i,reg} and its
factor L_i (eq. localdualoperatorwithU); fill-reducing ordering.
Readings of what the paper leaves open (element type, regularisation, gluing, ordering) are
listed in DESIGN.md §3 and SURVEY.md §8.3 items 2-6.
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")


def build_lib(force: bool = False) -> str:
    """Compile synth/csrc/chol.c into synth/libsynth.so (gcc, host only)."""
    src = os.path.join(_HERE, "csrc", "chol.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


@functools.lru_cache(maxsize=1)
def _lib():
    lib = ctypes.CDLL(build_lib())
    lib.synth_cholesky.restype = ctypes.c_int
    lib.synth_cholesky.argtypes = [
        ctypes.c_int32,
        ctypes.c_void_p,
        ctypes.c_void_p,
        ctypes.c_void_p,
        ctypes.c_void_p,
        ctypes.c_void_p,
        ctypes.c_void_p,
        ctypes.POINTER(ctypes.c_int64),
    ]
    return lib


def sparse_cholesky(C: sp.spmatrix):
    """L (CSC, diagonal first, rows ascending) with C = L L^T; C symmetric positive definite."""
    C = sp.csc_matrix(C)
    C.sort_indices()
    n = C.shape[0]
    Ap = np.ascontiguousarray(C.indptr, dtype=np.int64)
    Ai = np.ascontiguousarray(C.indices, dtype=np.int32)
    Ax = np.ascontiguousarray(C.data, dtype=np.float64)
    Lp = np.zeros(n + 1, dtype=np.int64)
    nnz = ctypes.c_int64(0)
    lib = _lib()
    rc = lib.synth_cholesky(n, Ap.ctypes.data, Ai.ctypes.data, Ax.ctypes.data, Lp.ctypes.data, None, None,
                            ctypes.byref(nnz))
    Li = np.zeros(nnz.value, dtype=np.int32)
    Lx = np.zeros(nnz.value, dtype=np.float64)
    rc = lib.synth_cholesky(n, Ap.ctypes.data, Ai.ctypes.data, Ax.ctypes.data, Lp.ctypes.data, Li.ctypes.data,
                            Lx.ctypes.data, ctypes.byref(nnz))
    if rc != 0:
        raise ValueError(f"sparse_cholesky: non-positive pivot at column {rc - 1}")
    return Lp, Li, Lx


# ----------------------------------------------------------------------------------------------
# Q1 element matrices (2-point Gauss per axis on [0,h]^d)
# ----------------------------------------------------------------------------------------------

def _q1_shape_grads(d: int, xi: np.ndarray, h: float) -> np.ndarray:
    """Gradients (2^d x d) of the lexicographic (x fastest) Q1 shape functions at point xi in [0,1]^d."""
    nn = 2 ** d
    g = np.zeros((nn, d))
    for a in range(nn):
        bits = [(a >> k) & 1 for k in range(d)]
        for k in range(d):
            v = 1.0
            for l in range(d):
                if l == k:
                    v *= 1.0 if bits[l] else -1.0
                else:
                    v *= xi[l] if bits[l] else 1.0 - xi[l]
            g[a, k] = v / h
    return g


@functools.lru_cache(maxsize=16)
def element_matrix(d: int, physics: str, h: float = 1.0, young: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """Q1 element stiffness for unit coefficient; local DOF = local_node*dpn + component."""
    gp = np.array([(1 - 1 / np.sqrt(3)) / 2, (1 + 1 / np.sqrt(3)) / 2])
    w = 0.5 ** d * h ** d
    nn = 2 ** d
    if physics == "heat":
        K = np.zeros((nn, nn))
        for idx in np.ndindex(*([2] * d)):
            G = _q1_shape_grads(d, gp[list(idx)], h)
            K += w * G @ G.T
        return K
    if physics == "elasticity":
        assert d == 3, "elasticity fixtures are 3D"
        lam = young * nu / ((1 + nu) * (1 - 2 * nu))
        mu = young / (2 * (1 + nu))
        D = np.zeros((6, 6))
        D[:3, :3] = lam
        D[np.arange(3), np.arange(3)] += 2 * mu
        D[3, 3] = D[4, 4] = D[5, 5] = mu
        K = np.zeros((3 * nn, 3 * nn))
        for idx in np.ndindex(2, 2, 2):
            G = _q1_shape_grads(3, gp[list(idx)], h)
            B = np.zeros((6, 3 * nn))
            for a in range(nn):
                gx, gy, gz = G[a]
                B[0, 3 * a + 0] = gx
                B[1, 3 * a + 1] = gy
                B[2, 3 * a + 2] = gz
                B[3, 3 * a + 1] = gz
                B[3, 3 * a + 2] = gy
                B[4, 3 * a + 0] = gz
                B[4, 3 * a + 2] = gx
                B[5, 3 * a + 0] = gy
                B[5, 3 * a + 1] = gx
            K += w * B.T @ D @ B
        return K
    raise ValueError(physics)


def _element_connectivity(d: int, E: int) -> np.ndarray:
    """(E^d, 2^d) local node ids of each element, lexicographic (x fastest) in both."""
    N = E + 1
    grids = np.meshgrid(*([np.arange(E)] * d), indexing="ij")
    # element coordinates with x fastest: grids[k] has axis k index; flatten in (z,y,x) order
    coords = [g.transpose(*reversed(range(d))).ravel() for g in grids]
    conn = np.zeros((E ** d, 2 ** d), dtype=np.int64)
    for a in range(2 ** d):
        node = np.zeros(E ** d, dtype=np.int64)
        stride = 1
        for k in range(d):
            node += (coords[k] + ((a >> k) & 1)) * stride
            stride *= N
        conn[:, a] = node
    return conn


def assemble_subdomain(d: int, E: int, physics: str, elem_coef: Optional[np.ndarray], h: float) -> sp.csr_matrix:
    """Unregularised subdomain stiffness K_i (natural lexicographic node order, DOF = node*dpn+c)."""
    dpn = 1 if physics == "heat" else 3
    Ke = element_matrix(d, physics, h)
    conn = _element_connectivity(d, E)
    dofs = (conn[:, :, None] * dpn + np.arange(dpn)[None, None, :]).reshape(conn.shape[0], -1)
    ne, nd = dofs.shape
    rows = np.repeat(dofs, nd, axis=1).ravel()
    cols = np.tile(dofs, (1, nd)).ravel()
    coef = np.ones(ne) if elem_coef is None else elem_coef
    vals = (coef[:, None, None] * Ke[None, :, :]).ravel()
    n = (E + 1) ** d * dpn
    K = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    K.sum_duplicates()
    # exactly symmetric with a symmetric stored pattern (the union of both triangles; sums that cancel
    # to round-off stay stored, as in a connectivity-based FEM pattern), so every consumer (oracle,
    # host factor, device factorization) sees the same matrix whichever triangle it reads
    K = ((K + K.T) * 0.5).tocsr()
    K.sort_indices()
    return K


def fixing_dofs(d: int, E: int, physics: str) -> np.ndarray:
    """DOFs held by the regularising springs (SURVEY §8.3 reading 2)."""
    N = E + 1
    if physics == "heat":
        return np.array([0], dtype=np.int64)
    A, B, C = 0, N - 1, (N - 1) * N
    return np.array([3 * A + 0, 3 * A + 1, 3 * A + 2, 3 * B + 1, 3 * B + 2, 3 * C + 2], dtype=np.int64)


def regularize(K: sp.csr_matrix, fix: np.ndarray) -> sp.csr_matrix:
    """K_reg = K + rho * sum_f e_f e_f^T with rho = mean(diag K) (pattern unchanged: diagonal exists)."""
    rho = float(K.diagonal().mean())
    D = sp.coo_matrix((np.full(len(fix), rho), (fix, fix)), shape=K.shape)
    Kr = (K + D).tocsr()
    Kr.sort_indices()
    return Kr


# ----------------------------------------------------------------------------------------------
# geometric nested dissection (SURVEY §8.3 reading 6)
# ----------------------------------------------------------------------------------------------

def nested_dissection_nodes(d: int, N: int, rng: Optional[np.random.Generator] = None) -> np.ndarray:
    """new->old node order on an N^d lexicographic grid: split the longest axis at its middle plane,
    order (left, right, separator); boxes with <= 2 nodes per axis stay in natural order.  With `rng`
    (perturbed patterns, one ordering per subdomain like a graph partitioner's): the split plane is
    jittered by -1/0/+1 and ties between equally long axes are broken at random."""
    out: List[np.ndarray] = []

    def natural(lo, hi):
        rng = [np.arange(lo[k], hi[k]) for k in range(d)]
        g = np.meshgrid(*rng, indexing="ij")
        idx = np.zeros(g[0].shape, dtype=np.int64)
        stride = 1
        for k in range(d):
            idx = idx + g[k] * stride
            stride *= N
        return idx.transpose(*reversed(range(d))).ravel()

    def rec(lo, hi):
        ext = [hi[k] - lo[k] for k in range(d)]
        if min(ext) <= 0:
            return
        if max(ext) <= 2:
            out.append(natural(lo, hi))
            return
        if rng is None:
            ax = max(range(d), key=lambda k: (ext[k], k))
            mid = lo[ax] + ext[ax] // 2
        else:
            longest = [k for k in range(d) if ext[k] == max(ext)]
            ax = int(longest[rng.integers(len(longest))])
            mid = lo[ax] + ext[ax] // 2 + (int(rng.integers(-1, 2)) if ext[ax] >= 5 else 0)
        lhi = list(hi)
        lhi[ax] = mid
        rlo = list(lo)
        rlo[ax] = mid + 1
        slo = list(lo)
        slo[ax] = mid
        shi = list(hi)
        shi[ax] = mid + 1
        rec(lo, lhi)
        rec(rlo, hi)
        out.append(natural(slo, shi))

    rec([0] * d, [N] * d)
    order = np.concatenate(out)
    assert len(order) == N ** d and len(np.unique(order)) == N ** d
    return order


# ----------------------------------------------------------------------------------------------
# problem container
# ----------------------------------------------------------------------------------------------

@dataclass
class Subdomain:
    id: int
    n: int
    kappa: float
    perm: np.ndarray            # int32, perm[new] = old DOF (fill-reducing)
    L_colptr: np.ndarray        # int64 (n+1), CSC of L, diagonal first, rows ascending
    L_rowidx: np.ndarray        # int32
    Bt_colptr: np.ndarray       # int32 (m+1), CSC of B~^T, rows in ORIGINAL dof numbering
    Bt_rowidx: np.ndarray       # int32
    Bt_values: np.ndarray       # float64
    lambda_map: np.ndarray      # int64 (m), local -> global multiplier id
    _K_ref: sp.csr_matrix = field(repr=False, default=None)
    _L_ref_values: np.ndarray = field(repr=False, default=None)
    _K_own: Optional[sp.csr_matrix] = field(repr=False, default=None)
    _L_own: Optional[np.ndarray] = field(repr=False, default=None)

    @property
    def m(self) -> int:
        return len(self.Bt_colptr) - 1

    @property
    def K_reg(self) -> sp.csr_matrix:
        """Regularised stiffness in the natural DOF order (the oracle's input)."""
        if self._K_own is not None:
            return self._K_own
        return (self._K_ref * self.kappa).tocsr()

    @property
    def L_values(self) -> np.ndarray:
        """Values of L (CSC order) with P K_reg P^T = L L^T (the GPU path's input)."""
        if self._L_own is not None:
            return self._L_own
        return self._L_ref_values * np.sqrt(self.kappa)

    def K_lower(self):
        """(colptr int64, rowidx int32, values float64): CSC of the lower triangle of K_reg in the
        natural DOF order -- the input of the device factorization (sc_factor_attach / factorize)."""
        T = sp.tril(self.K_reg).tocsc()
        T.sort_indices()
        return (np.ascontiguousarray(T.indptr, dtype=np.int64), np.ascontiguousarray(T.indices, dtype=np.int32),
                np.ascontiguousarray(T.data, dtype=np.float64))

    def Bt_dense(self) -> np.ndarray:
        Bt = np.zeros((self.n, self.m))
        for j in range(self.m):
            for p in range(self.Bt_colptr[j], self.Bt_colptr[j + 1]):
                Bt[self.Bt_rowidx[p], j] += self.Bt_values[p]
        return Bt

    def Bt_sparse(self) -> sp.csc_matrix:
        return sp.csc_matrix((self.Bt_values, self.Bt_rowidx, self.Bt_colptr), shape=(self.n, self.m))


@dataclass
class Problem:
    name: str
    dim: int
    physics: str
    S: int
    E: int
    subdomains: List[Subdomain]
    n_lambda: int

    def __len__(self):
        return len(self.subdomains)


def _glue(d: int, S: int, E: int, dpn: int, redundant: bool, dirichlet: bool):
    """Multipliers: (subdomain, local dof, global id, value) arrays, sorted by (subdomain, global id).

    Gluing (SURVEY §8.3 readings 3-4): for a node shared by subdomains s_0<...<s_k, non-redundant
    gluing puts one multiplier per component on each consecutive pair (s_a, s_{a+1}) with +1 in s_a
    and -1 in s_{a+1}; redundant gluing uses every pair.  Dirichlet on the global x=0 face: one +1
    multiplier per component for every subdomain copy of the node.
    """
    NG = S * E + 1
    N = E + 1
    g = np.indices([NG] * d).reshape(d, -1)[::-1]  # g[k] = coordinate along axis k, x fastest
    # candidate subdomain index along each axis: lower and upper (equal when not on an interface)
    lo = np.minimum(g // E, S - 1)
    on_if = (g % E == 0) & (g > 0) & (g < S * E)
    lo = np.where(on_if, g // E - 1, lo)
    hi = np.where(on_if, g // E, lo)
    nshare = np.prod(np.where(on_if, 2, 1), axis=0)
    on_x0 = g[0] == 0
    keep = (nshare >= 2) | (on_x0 if dirichlet else False)
    gk, lok, hik = g[:, keep], lo[:, keep], hi[:, keep]
    node_ids = np.nonzero(keep)[0]
    nk = gk.shape[1]
    # enumerate up to 2^d sharing subdomains (duplicates when lo == hi)
    subs = np.zeros((nk, 2 ** d), dtype=np.int64)
    locs = np.zeros((nk, 2 ** d), dtype=np.int64)
    for c in range(2 ** d):
        sid = np.zeros(nk, dtype=np.int64)
        lid = np.zeros(nk, dtype=np.int64)
        sstride, lstride = 1, 1
        for k in range(d):
            sk = np.where((c >> k) & 1, hik[k], lok[k])
            sid += sk * sstride
            lid += (gk[k] - sk * E) * lstride
            sstride *= S
            lstride *= N
        subs[:, c] = sid
        locs[:, c] = lid
    order = np.argsort(subs, axis=1, kind="stable")
    subs = np.take_along_axis(subs, order, axis=1)
    locs = np.take_along_axis(locs, order, axis=1)
    # unique per row
    dup = np.zeros_like(subs, dtype=bool)
    dup[:, 1:] = subs[:, 1:] == subs[:, :-1]
    out_s, out_l, out_key, out_v = [], [], [], []
    key_base = node_ids.astype(np.int64) * 256
    # compact each row's unique subdomains to the left
    cnt = (~dup).sum(axis=1)
    pos = np.cumsum(~dup, axis=1) - 1
    U_s = np.full_like(subs, -1)
    U_l = np.full_like(locs, -1)
    rr, cc = np.nonzero(~dup)
    U_s[rr, pos[rr, cc]] = subs[rr, cc]
    U_l[rr, pos[rr, cc]] = locs[rr, cc]
    slot = 0
    maxc = 2 ** d
    pairs = [(a, a + 1) for a in range(maxc - 1)] if not redundant else [(a, b) for a in range(maxc) for b in range(a + 1, maxc)]
    for (a, b) in pairs:
        sel = cnt > b
        idx = np.nonzero(sel)[0]
        for comp in range(dpn):
            key = key_base[idx] + slot
            out_s += [U_s[idx, a], U_s[idx, b]]
            out_l += [U_l[idx, a] * dpn + comp, U_l[idx, b] * dpn + comp]
            out_key += [key, key]
            out_v += [np.ones(len(idx)), -np.ones(len(idx))]
            slot += 1
    if dirichlet:
        x0 = gk[0] == 0
        for a in range(maxc):
            sel = x0 & (cnt > a)
            idx = np.nonzero(sel)[0]
            for comp in range(dpn):
                key = key_base[idx] + slot
                out_s.append(U_s[idx, a])
                out_l.append(U_l[idx, a] * dpn + comp)
                out_key.append(key)
                out_v.append(np.ones(len(idx)))
                slot += 1
    assert slot < 256
    s_all = np.concatenate(out_s)
    l_all = np.concatenate(out_l)
    k_all = np.concatenate(out_key)
    v_all = np.concatenate(out_v)
    uk, gid = np.unique(k_all, return_inverse=True)
    o = np.lexsort((gid, s_all))
    return s_all[o], l_all[o], gid[o].astype(np.int64), v_all[o], len(uk)


def make_problem(dim: int, physics: str, S: int, E: int, *, seed: int = 0, coef: str = "subdomain",
                 redundant: bool = False, dirichlet: bool = True, subdomains: Optional[List[int]] = None,
                 name: str = "", perturbed: bool = False) -> Problem:
    """Build a structured FETI problem (see module docstring).  `subdomains` restricts which
    subdomains get materialised (the gluing is always that of the full decomposition)."""
    assert physics in ("heat", "elasticity")
    dpn = 1 if physics == "heat" else 3
    N = E + 1
    h = 1.0 / (S * E)
    nsub_total = S ** dim
    ids = list(range(nsub_total)) if subdomains is None else list(subdomains)
    s_all, l_all, g_all, v_all, n_lambda = _glue(dim, S, E, dpn, redundant, dirichlet)
    starts = np.searchsorted(s_all, np.arange(nsub_total + 1))

    fix = fixing_dofs(dim, E, physics)
    node_order = nested_dissection_nodes(dim, N)
    perm = (node_order[:, None] * dpn + np.arange(dpn)[None, :]).ravel().astype(np.int32)
    n = N ** dim * dpn

    K_ref = L_ref = None
    if coef == "subdomain" and not perturbed:
        K_ref = regularize(assemble_subdomain(dim, E, physics, None, h), fix)
        C = K_ref[perm][:, perm]
        Lp, Li, Lx_ref = sparse_cholesky(C)
    if perturbed and K_ref is None:
        K_ref = regularize(assemble_subdomain(dim, E, physics, None, h), fix)

    def one(i):
        rng = np.random.default_rng([seed, i])
        kappa = float(rng.uniform(1.0, 10.0))
        a, b = starts[i], starts[i + 1]
        m = b - a
        Bt_colptr = np.arange(m + 1, dtype=np.int32)
        Bt_rowidx = l_all[a:b].astype(np.int32)
        Bt_values = v_all[a:b].astype(np.float64)
        lam = g_all[a:b].astype(np.int64)
        if coef == "subdomain" and not perturbed:
            sd = Subdomain(i, n, kappa, perm, Lp, Li, Bt_colptr, Bt_rowidx, Bt_values, lam,
                           _K_ref=K_ref, _L_ref_values=Lx_ref)
        elif perturbed:
            # a distinct fill-reducing ordering (hence L pattern) per subdomain, same K
            no = nested_dissection_nodes(dim, N, np.random.default_rng([seed, i, 7]))
            perm_i = (no[:, None] * dpn + np.arange(dpn)[None, :]).ravel().astype(np.int32)
            K = (K_ref * kappa).tocsr()
            Lp_i, Li_i, Lx_i = sparse_cholesky(K[perm_i][:, perm_i])
            sd = Subdomain(i, n, 1.0, perm_i, Lp_i, Li_i, Bt_colptr, Bt_rowidx, Bt_values, lam,
                           _K_own=K, _L_own=Lx_i)
        elif coef == "element":
            ec = rng.uniform(1.0, 10.0, size=E ** dim)
            K = regularize(assemble_subdomain(dim, E, physics, ec, h), fix)
            C = K[perm][:, perm]
            Lp_i, Li_i, Lx_i = sparse_cholesky(C)
            sd = Subdomain(i, n, 1.0, perm, Lp_i, Li_i, Bt_colptr, Bt_rowidx, Bt_values, lam,
                           _K_own=K, _L_own=Lx_i)
        else:
            raise ValueError(coef)
        return sd
    if perturbed or coef == "element":  # one host factorization per subdomain: in parallel
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=max(1, min(32, len(os.sched_getaffinity(0))))) as ex:
            subs: List[Subdomain] = list(ex.map(one, ids))
    else:
        subs = [one(i) for i in ids]
    return Problem(name or f"{dim}d-{physics}-S{S}-E{E}", dim, physics, S, E, subs, n_lambda)


# BASELINE.json configs (SURVEY §8.4 "Synthetic inputs, concrete")
CONFIGS: Dict[str, dict] = {
    "cfg1": dict(dim=2, physics="heat", S=4, E=8),
    "cfg2": dict(dim=2, physics="heat", S=32, E=64),
    "cfg3": dict(dim=3, physics="heat", S=8, E=16),
    "cfg4": dict(dim=3, physics="elasticity", S=8, E=12),
    "cfg5": dict(dim=3, physics="elasticity", S=4, E=24),
    # small parity/test configs (not bench lines)
    "t2d": dict(dim=2, physics="heat", S=3, E=6),
    "t3d": dict(dim=3, physics="heat", S=2, E=4),
    "t3e": dict(dim=3, physics="elasticity", S=2, E=3),
    # S=3 per axis: all 27 boundary classes (x=0 Dirichlet face / edges / corner, the other faces,
    # edges and corners, and the interior subdomain 13)
    "t3h3": dict(dim=3, physics="heat", S=3, E=4),
    "t3e3": dict(dim=3, physics="elasticity", S=3, E=3),
}


def config_problem(name: str, **kw) -> Problem:
    args = dict(CONFIGS[name])
    args.update(kw)
    return make_problem(name=name, **args)


def subdomain_K(problem: Problem, sd: Subdomain) -> sp.csr_matrix:
    """Unregularised K_i of a subdomain of a per-subdomain-coefficient problem (natural DOF order)."""
    h = 1.0 / (problem.S * problem.E)
    return (assemble_subdomain(problem.dim, problem.E, problem.physics, None, h) * sd.kappa).tocsr()


def kernel_basis(problem: Problem, sd: Subdomain) -> np.ndarray:
    """R_i: basis of ker K_i ("R_i containing the basis vectors of Ker K_i") in the
    natural DOF order: constants for heat, the 6 rigid-body modes (3 translations, 3 rotations
    about the subdomain's corner) for elasticity."""
    N = problem.E + 1
    d = problem.dim
    if problem.physics == "heat":
        return np.ones((sd.n, 1))
    g = np.indices([N] * d).reshape(d, -1)[::-1].astype(np.float64)  # g[k] = coordinate along axis k, x fastest
    x, y, z = g[0], g[1], g[2]
    R = np.zeros((sd.n, 6))
    for c in range(3):
        R[c::3, c] = 1.0
    R[0::3, 3], R[1::3, 3] = -y, x       # rotation about z
    R[1::3, 4], R[2::3, 4] = -z, y       # rotation about x
    R[0::3, 5], R[2::3, 5] = z, -x       # rotation about y
    return R


def chain_1d_problem(n: int) -> Problem:
    """1D chain K = tridiag(-1,2,-1) (SPD without regularisation), B~^T = [e_1, e_n], identity
    ordering.  Closed form F = [[n,1],[1,n]]/(n+1) (SURVEY §8.3 pins)."""
    main = np.full(n, 2.0)
    off = np.full(n - 1, -1.0)
    K = sp.diags([off, main, off], [-1, 0, 1], format="csr")
    perm = np.arange(n, dtype=np.int32)
    Lp, Li, Lx = sparse_cholesky(K)
    Bt_colptr = np.array([0, 1, 2], dtype=np.int32)
    Bt_rowidx = np.array([0, n - 1], dtype=np.int32)
    Bt_values = np.array([1.0, 1.0])
    sd = Subdomain(0, n, 1.0, perm, Lp, Li, Bt_colptr, Bt_rowidx, Bt_values, np.array([0, 1], dtype=np.int64),
                   _K_own=K, _L_own=Lx)
    return Problem(f"chain{n}", 1, "heat", 1, n - 1, [sd], 2)


def custom_problem(K: sp.spmatrix, Bt: np.ndarray, perm: Optional[np.ndarray] = None, name: str = "custom") -> Problem:
    """One subdomain from an explicit SPD K (natural order) and a dense B~^T (n x m)."""
    K = sp.csr_matrix(K)
    n = K.shape[0]
    perm = np.arange(n, dtype=np.int32) if perm is None else np.asarray(perm, dtype=np.int32)
    C = K[perm][:, perm]
    Lp, Li, Lx = sparse_cholesky(C)
    Bt = np.asarray(Bt, dtype=np.float64)
    B = sp.csc_matrix(Bt)
    B.sort_indices()
    m = Bt.shape[1]
    sd = Subdomain(0, n, 1.0, perm, Lp, Li, B.indptr.astype(np.int32), B.indices.astype(np.int32),
                   B.data.astype(np.float64), np.arange(m, dtype=np.int64), _K_own=K, _L_own=Lx)
    return Problem(name, 0, "custom", 1, 0, [sd], m)
