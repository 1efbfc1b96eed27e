"""Pins for the CPU oracle (oracle/): checks against what the paper and mathematics fix, never
against the oracle's own formula retyped.  Runs on CPU (-m "not gpu").

Pins: SPEC hand cases (tests/golden/hand_cases.json, cited per case), the 1D closed form, a
brute-force dense inverse (LU via numpy, a different route from the oracle's band Cholesky),
the Schur-complement identity K^-1[b,b] = (K_bb - K_bi K_ii^-1 K_ib)^-1, an independent sparse
LU (SuperLU) for F*lambda, symmetry / PSD invariants and the additivity of local operators
into the global B K^+ B^T ("can be combined additively").
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from synth import chain_1d_problem, make_problem

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_cases.json")))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# ---------------------------------------------------------------- hand cases (golden, cited)

def test_cholesky_hand_case():
    c = GOLD["cholesky_2x2"]
    L = oracle.cholesky(sp.csr_matrix(np.array(c["K"], dtype=float)))
    np.testing.assert_array_equal(L, np.array(c["L"], dtype=float))


@pytest.mark.parametrize("case,fn", [("trsv_forward", "forward"), ("factor_split_block", "forward"),
                                     ("trsv_backward", "backward")])
def test_triangular_solve_hand_cases(case, fn):
    c = GOLD[case]
    x = getattr(oracle, fn)(np.array(c["L"], dtype=float), np.array(c["b"], dtype=float))
    np.testing.assert_array_equal(x, np.array(c["x"], dtype=float))


def test_trsm_hand_case_columnwise():
    c = GOLD["trsm_2rhs"]
    L = np.array(c["L"], dtype=float)
    X = np.array(c["X"], dtype=float)
    Y = np.stack([oracle.forward(L, X[:, j]) for j in range(X.shape[1])], axis=1)
    np.testing.assert_array_equal(Y, np.array(c["Y"], dtype=float))


@pytest.mark.parametrize("case", ["assembly_K2I", "chain_n3"])
def test_dual_operator_hand_cases(case):
    c = GOLD[case]
    F = oracle.dual_operator(sp.csr_matrix(np.array(c["K"], dtype=float)), np.array(c["Bt"], dtype=float))
    np.testing.assert_allclose(F, np.array(c["F"], dtype=float), rtol=0, atol=1e-15)


def test_identity_K_gives_BBt():
    """K = I -> F = B B^T, for a general (not Boolean, multi-nonzero) B."""
    rng = np.random.default_rng(3)
    n, m = 17, 9
    Bt = rng.standard_normal((n, m)) * (rng.random((n, m)) < 0.3)
    F = oracle.dual_operator(sp.identity(n, format="csr"), Bt)
    np.testing.assert_allclose(F, Bt.T @ Bt, rtol=1e-14, atol=1e-14)


# ---------------------------------------------------------------- closed form

@pytest.mark.parametrize("n", [3, 7, 50, 513])
def test_chain_closed_form(n):
    P = chain_1d_problem(n)
    F = oracle.subdomain_F(P.subdomains[0])
    exact = np.array([[n, 1.0], [1.0, n]]) / (n + 1)
    # cond(K) grows like n^2; compare entrywise against the largest entry
    np.testing.assert_allclose(F, exact, rtol=0, atol=1e-13 * exact.max())


# ---------------------------------------------------------------- brute force (dense inverse)

SMALL = [
    dict(dim=2, physics="heat", S=2, E=2),
    dict(dim=3, physics="heat", S=2, E=2),
    dict(dim=3, physics="elasticity", S=2, E=2),
    dict(dim=2, physics="heat", S=4, E=8),        # the cfg1 mesh itself (n=81)
    dict(dim=2, physics="heat", S=3, E=5, coef="element"),
    dict(dim=3, physics="elasticity", S=2, E=2, coef="element", redundant=True),
]


@pytest.mark.parametrize("spec", SMALL, ids=lambda s: "-".join(str(v) for v in s.values()))
def test_bruteforce_inverse(spec):
    P = make_problem(**spec)
    for sd in P.subdomains[:4]:
        K = sd.K_reg.toarray()
        Bt = sd.Bt_dense()
        F_brute = Bt.T @ np.linalg.inv(K) @ Bt
        F = oracle.subdomain_F(sd)
        assert rel(F, F_brute) < 1e-12


def test_bruteforce_random_spd_general_B():
    """Non-symmetric-looking, multi-nonzero B~ with general values: a transposed operand, a wrong
    sign or a dropped term in O3/O4 would show here."""
    rng = np.random.default_rng(11)
    n, m = 40, 13
    A = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.15)
    K = A @ A.T + n * np.eye(n)
    K[np.abs(K) < 1e-300] = 0
    Bt = rng.standard_normal((n, m)) * (rng.random((n, m)) < 0.2)
    Bt[rng.integers(0, n, m), np.arange(m)] = rng.uniform(-3, 3, m)
    F = oracle.dual_operator(sp.csr_matrix(K), Bt)
    assert rel(F, Bt.T @ np.linalg.solve(K, Bt)) < 1e-12
    # dense triangular factor reproduces K
    L = oracle.cholesky(sp.csr_matrix(K))
    assert np.allclose(np.triu(L, 1), 0)
    assert rel(L @ L.T, K) < 1e-14


# ---------------------------------------------------------------- Schur identity (independent route)

@pytest.mark.parametrize("spec", [dict(dim=2, physics="heat", S=3, E=6), dict(dim=3, physics="heat", S=2, E=4),
                                  dict(dim=3, physics="elasticity", S=2, E=3)])
def test_schur_identity(spec):
    P = make_problem(**spec)
    sd = P.subdomains[-1]
    K = sd.K_reg.toarray()
    Bt = sd.Bt_sparse().tocsc()
    d = np.array([Bt.indices[Bt.indptr[j]] for j in range(sd.m)])  # one nonzero per column here
    s = np.array([Bt.data[Bt.indptr[j]] for j in range(sd.m)])
    b = np.unique(d)
    i = np.setdiff1d(np.arange(sd.n), b)
    S = K[np.ix_(b, b)] - K[np.ix_(b, i)] @ np.linalg.solve(K[np.ix_(i, i)], K[np.ix_(i, b)])
    Kinv_bb = np.linalg.inv(S)
    pos = np.searchsorted(b, d)
    F_schur = (s[:, None] * Kinv_bb[np.ix_(pos, pos)]) * s[None, :]
    F = oracle.subdomain_F(sd)
    assert rel(F, F_schur) < 1e-12


# ---------------------------------------------------------------- invariants

def test_invariants_symmetry_psd_apply():
    P = make_problem(dim=3, physics="elasticity", S=2, E=3, coef="element")
    rng = np.random.default_rng(5)
    for sd in P.subdomains[:3]:
        F = oracle.subdomain_F(sd)
        assert np.linalg.norm(F - F.T) / np.linalg.norm(F) < 1e-14
        ev = np.linalg.eigvalsh(0.5 * (F + F.T))
        assert ev.min() >= -1e-10 * ev.max()
        # F lambda = B K^-1 (B^T lambda) through SuperLU (independent solver)
        lam = rng.standard_normal(sd.m)
        Bt = sd.Bt_sparse()
        q = Bt.T @ spla.spsolve(sd.K_reg.tocsc(), Bt @ lam)
        assert rel(F @ lam, q) < 1e-12


def test_column_sampling_matches_full():
    P = make_problem(dim=2, physics="heat", S=3, E=6)
    sd = P.subdomains[4]
    F = oracle.subdomain_F(sd)
    cols = [0, 5, sd.m - 1, 3]
    np.testing.assert_array_equal(oracle.subdomain_F(sd, cols), F[:, cols])


def test_not_spd_raises():
    K = sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(oracle.OracleError):
        oracle.dual_operator(K, np.eye(2))


def test_additivity_global_operator():
    """sum_i scatter(F_i) = B K^+ B^T of the whole block system."""
    P = make_problem(dim=2, physics="heat", S=2, E=3)
    M = P.n_lambda
    F_sum = np.zeros((M, M))
    blocks, Bcols = [], []
    for sd in P.subdomains:
        F = oracle.subdomain_F(sd)
        idx = sd.lambda_map
        F_sum[np.ix_(idx, idx)] += F
        blocks.append(sd.K_reg.toarray())
        Bl = np.zeros((M, sd.n))
        Bl[idx, :] = sd.Bt_dense().T
        Bcols.append(Bl)
    Kg = np.zeros((sum(b.shape[0] for b in blocks),) * 2)
    o = 0
    for b in blocks:
        Kg[o:o + b.shape[0], o:o + b.shape[0]] = b
        o += b.shape[0]
    B = np.hstack(Bcols)
    F_glob = B @ np.linalg.inv(Kg) @ B.T
    assert rel(F_sum, F_glob) < 1e-12
