"""Device numeric factorization (§2.2 two-stage factorization).

The factor L of P K_reg P^T is unique (K_reg SPD), so the device L is compared entry by entry with
the oracle's Cholesky (oracle.cholesky: textbook band Cholesky, pinned in test_oracle_pins.py) of the
permuted K_reg at small sizes, and with the input generator's own sparse factor (synth/csrc/chol.c,
an independent up-looking code) at full size; F assembled from the device L is compared with the
oracle's F (which never sees L).  CPU tests cover the symbolic stage on host-only plans.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg  # noqa: F401

import oracle
from paper_2509_21037_b200 import SCPlan, ScError
from paper_2509_21037_b200 import sc as scmod
from synth import config_problem, make_problem

TOL = 1e-10
TOL_L = 1e-10  # L entries relative to max|L|: the north_star's FP64 bar applied to the factor; the
               # rigorous check is the backward error below (two FP64 factorizations that differ only
               # in summation order agree to ~1e-12 here)
U = 2.0 ** -53


def assert_backward_stable(sd, Lx):
    """Normwise backward error of the computed factor: ||L L^T - A||_F <= c (3c + 1) u ||A||_F with c
    the largest column count of L (Higham, Accuracy and Stability, Thm 10.4, with the inner-product
    length n of the dense bound replaced by the column count of the sparse factor).  The device path
    solves the rows below each diagonal block with the block's explicit inverse, which is normwise
    (not componentwise) stable, so the check is normwise."""
    n = sd.n
    L = sp.csc_matrix((Lx, sd.L_rowidx, sd.L_colptr), shape=(n, n))
    A = sd.K_reg[sd.perm][:, sd.perm]
    c = int(np.diff(sd.L_colptr).max())
    res = sp.linalg.norm(L @ L.T - A) / sp.linalg.norm(A)
    assert res <= c * (3 * c + 1) * U, (res, c)
    return res


def _torch():
    import torch
    return torch


def K_patterns(subs):
    return [sd.K_lower()[:2] for sd in subs]


def K_dev(subs):
    torch = _torch()
    return [torch.from_numpy(sd.K_lower()[2]).cuda() for sd in subs]


def L_out(subs, dtype=None):
    torch = _torch()
    return [torch.zeros(int(sd.L_colptr[-1]), dtype=dtype or torch.float64, device="cuda") for sd in subs]


def dense_L(sd, Lx):
    n = sd.n
    cols = np.repeat(np.arange(n), np.diff(sd.L_colptr))
    L = np.zeros((n, n))
    L[sd.L_rowidx, cols] = Lx
    return L


def assert_parity(F_gpu, F_ref, tol=TOL):
    nrm = np.linalg.norm(F_ref)
    rel = np.linalg.norm(F_gpu - F_ref) / nrm
    assert rel <= tol, f"relative Frobenius error {rel:.3e} > {tol}"
    assert np.abs(F_gpu - F_ref).max() <= tol * np.abs(F_ref).max()


# ------------------------------------------------------------------ CPU: symbolic stage (host-only plan)

def test_factor_symbolic_host_only_stats():
    """Host-only plan: sc_factor_attach runs the symbolic stage; flops_factor_useful = sum_k cc_k^2
    (column counts of L), the textbook Cholesky count; K_nnz bytes; levels/tasks populated."""
    P = config_problem("t3e")
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1)
    plan.factor_attach(K_patterns(P.subdomains))
    st = plan.stats()
    want = sum(float((np.diff(sd.L_colptr).astype(float) ** 2).sum()) for sd in P.subdomains)
    assert st["flops_factor_useful"] == pytest.approx(want, rel=1e-12)
    assert st["bytes_K_values"] == 8 * sum(int(sd.K_lower()[0][-1]) for sd in P.subdomains)
    assert st["factor_tasks"] > 0 and st["factor_panels"] > 0 and st["factor_max_level"] >= 1
    assert st["flops_factor_executed"] >= 0.5 * st["flops_factor_useful"]
    with pytest.raises(ScError) as e:
        plan.factorize([0] * plan.nsub, [0] * plan.nsub, stream=0)
    assert e.value.status == scmod.SC_ERR_STATE


def test_factor_symbolic_rejects_K_outside_L():
    """A K entry whose permuted position is not in the pattern of L is a pattern error."""
    P = config_problem("cfg1")
    sd = P.subdomains[0]
    plan = SCPlan([sd], n_lambda=P.n_lambda, device=-1)
    cp, ri, _ = sd.K_lower()
    iperm = np.argsort(sd.perm)
    Ld = np.zeros((sd.n, sd.n), dtype=bool)
    Ld[sd.L_rowidx, np.repeat(np.arange(sd.n), np.diff(sd.L_colptr))] = True
    # find an (i, j), i > j, whose permuted position is outside L, and add it to K's pattern
    bad = None
    for j in range(sd.n):
        for i in range(j + 1, sd.n):
            r, c = max(iperm[i], iperm[j]), min(iperm[i], iperm[j])
            if not Ld[r, c]:
                bad = (i, j)
                break
        if bad:
            break
    assert bad is not None
    K = sp.csc_matrix((np.ones(len(ri)), ri, cp), shape=(sd.n, sd.n)).tolil()
    K[bad[0], bad[1]] = 1.0
    K = K.tocsc()
    K.sort_indices()
    with pytest.raises(ScError) as e:
        plan.factor_attach([(K.indptr, K.indices)])
    assert e.value.status == scmod.SC_ERR_PATTERN


def test_factor_symbolic_rejects_upper_and_mismatched_class():
    P = config_problem("cfg1")
    subs = P.subdomains[:2]
    plan = SCPlan(subs, n_lambda=P.n_lambda, device=-1)
    cp, ri, _ = subs[0].K_lower()
    K = sp.csc_matrix((np.ones(len(ri)), ri, cp), shape=(subs[0].n,) * 2)
    U = K.T.tocsc()
    U.sort_indices()
    with pytest.raises(ScError) as e:  # upper triangle given
        plan.factor_attach([(U.indptr, U.indices)] * 2)
    assert e.value.status == scmod.SC_ERR_PATTERN
    if plan.stats()["n_classes"] == 1:  # both subdomains in one class: K patterns must agree
        D = sp.diags(np.ones(subs[0].n)).tocsc()
        with pytest.raises(ScError) as e:
            plan.factor_attach([(cp, ri), (D.indptr, D.indices)])
        assert e.value.status == scmod.SC_ERR_PATTERN


# ------------------------------------------------------------------ GPU: numeric stage

def _factorize(P, **kw):
    torch = _torch()
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, **kw)
    plan.factor_attach(K_patterns(P.subdomains))
    Kd = K_dev(P.subdomains)
    Lo = L_out(P.subdomains, dtype=torch.float32 if kw.get("precision") == 32 else None)
    plan.factorize(Kd, Lo)
    torch.cuda.synchronize()
    plan.check()
    return plan, Kd, Lo


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "t2d", "t3d", "t3e", "t3h3", "t3e3"])
def test_factor_matches_oracle_cholesky_and_F(cfg):
    """Device L == oracle Cholesky of P K_reg P^T (entry by entry, 1e-12 of max|L|; zeros off the
    pattern by construction of the CSC output), and F assembled from it == oracle F (1e-10)."""
    P = config_problem(cfg)
    plan, Kd, Lo = _factorize(P)
    for i, sd in enumerate(P.subdomains):
        C = sd.K_reg[sd.perm][:, sd.perm]
        Lref = oracle.cholesky(C)
        Ld = dense_L(sd, Lo[i].cpu().numpy())
        assert np.abs(Ld - Lref).max() <= TOL_L * np.abs(Lref).max()
        assert np.allclose(Lo[i].cpu().numpy(), sd.L_values, rtol=0, atol=TOL_L * np.abs(sd.L_values).max())
        assert_backward_stable(sd, Lo[i].cpu().numpy())
    plan.assemble(Lo)
    _torch().cuda.synchronize()
    plan.check()
    for i, sd in enumerate(P.subdomains):
        assert_parity(plan.get_F(i), oracle.subdomain_F(sd))


@pytest.mark.gpu
@pytest.mark.parametrize("spec", [dict(dim=2, physics="heat", S=3, E=5), dict(dim=3, physics="heat", S=2, E=3),
                                  dict(dim=3, physics="elasticity", S=2, E=2)])
def test_factor_heterogeneous_coefficients(spec):
    """Per-element coefficients: every subdomain has its own K values (and its own class)."""
    P = make_problem(coef="element", seed=3, **spec)
    plan, Kd, Lo = _factorize(P)
    for i, sd in enumerate(P.subdomains):
        Lref = oracle.cholesky(sd.K_reg[sd.perm][:, sd.perm])
        Ld = dense_L(sd, Lo[i].cpu().numpy())
        assert np.abs(Ld - Lref).max() <= TOL_L * np.abs(Lref).max()


@pytest.mark.gpu
def test_factor_deterministic_fp32_and_host_pipeline():
    """Bitwise determinism of two factorizations; precision 32 writes the FP64 result rounded to FP32;
    sc_factorize_assemble_host (H2D of K, chunked) gives bitwise the F of factorize + assemble."""
    torch = _torch()
    P = config_problem("t3h3")
    plan, Kd, Lo = _factorize(P)
    Lo2 = L_out(P.subdomains)
    plan.factorize(Kd, Lo2)
    torch.cuda.synchronize()
    for a, b in zip(Lo, Lo2):
        assert torch.equal(a, b)
    plan.assemble(Lo)
    torch.cuda.synchronize()
    F_dev = [plan.get_F(i) for i in range(plan.nsub)]
    for Kh in ([torch.from_numpy(sd.K_lower()[2]).pin_memory() for sd in P.subdomains],  # mapped gather
               [np.ascontiguousarray(sd.K_lower()[2]) for sd in P.subdomains]):             # pageable: memcpy
        plan.factorize_assemble_host(Kh)
        torch.cuda.synchronize()
        plan.check()
        for i in range(plan.nsub):
            assert np.array_equal(plan.get_F(i), F_dev[i])
    p32, _, L32 = _factorize(P, precision=32)
    for a, b in zip(L32, Lo):
        assert torch.equal(a, b.float())


@pytest.mark.gpu
def test_factor_zero_pivot_then_recovery():
    """A K that is not positive definite raises the sticky SC_ERR_ZERO_PIVOT for that subdomain;
    the next factorization with good values clears it."""
    torch = _torch()
    P = config_problem("cfg1")
    plan, Kd, Lo = _factorize(P)
    cp, ri, v = P.subdomains[5].K_lower()
    bad = v.copy()
    bad[cp[3]] = -1.0  # diagonal of DOF 3 (first entry of its lower column)
    Kbad = list(Kd)
    Kbad[5] = torch.from_numpy(bad).cuda()
    plan.factorize(Kbad, Lo)
    torch.cuda.synchronize()
    with pytest.raises(ScError) as e:
        plan.check()
    assert e.value.status == scmod.SC_ERR_ZERO_PIVOT
    plan.factorize(Kd, Lo)
    torch.cuda.synchronize()
    plan.check()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg2", "cfg3", "cfg4"])
def test_factor_full_size(cfg):
    """BASELINE configs at full size: device L against the input generator's independent sparse
    factor for every subdomain (max |diff| <= 1e-12 max|L|), and F of sampled subdomains/columns
    from the device L against the oracle (computed from K_reg, not from L)."""
    torch = _torch()
    P = config_problem(cfg)
    plan, Kd, Lo = _factorize(P)
    worst = 0.0
    for i, sd in enumerate(P.subdomains):
        ref = sd.L_values
        d = torch.from_numpy(ref).cuda()
        worst = max(worst, float((Lo[i] - d).abs().max() / d.abs().max()))
    assert worst <= TOL_L, worst
    for i in (0, len(P.subdomains) // 2, len(P.subdomains) - 1):
        assert_backward_stable(P.subdomains[i], Lo[i].cpu().numpy())
    plan.assemble(Lo)
    torch.cuda.synchronize()
    plan.check()
    rng = np.random.default_rng(5)
    for i in rng.choice(len(P.subdomains), 3, replace=False):
        sd = P.subdomains[int(i)]
        cols = sorted(set(rng.choice(sd.m, 8, replace=False).tolist()) | {0, sd.m - 1})
        assert_parity(plan.get_F(int(i))[:, cols], oracle.subdomain_F(sd, cols))
