"""Reference FETI dual problem for the PCPG tests (test infrastructure; uses the oracle's F_i).

PAPER.md P:200-254: R_i = basis of ker K_i, G = B R, e = R^T f, d = B K^+ f - c (c = 0), F = B K^+ B^T
(K_i^+ = K_{i,reg}^{-1}), and the dual problem [F -G; -G^T O][lambda; alpha] = [d; -e]
(eq. tfetidualproblem).  The reference solves it densely with numpy from the oracle's F_i; the
primal solution u_i = K_i^+ (f_i - B~_i^T lambda_i) + R_i alpha_i (eq. solutionUeval) is what the
pins check: gluing B u = 0 and equilibrium K_i u_i = f_i - B~_i^T lambda_i."""
import numpy as np
import scipy.sparse.linalg as spla

import oracle
from synth import kernel_basis, subdomain_K


def feti_data(P, seed=0):
    rng = np.random.default_rng(seed)
    subs = P.subdomains
    Rs = [kernel_basis(P, sd) for sd in subs]
    ks = [R.shape[1] for R in Rs]
    off = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
    nc = int(off[-1])
    fs = [rng.standard_normal(sd.n) for sd in subs]
    G = np.zeros((P.n_lambda, nc))
    d = np.zeros(P.n_lambda)
    e = np.zeros(nc)
    BR = []
    for i, sd in enumerate(subs):
        Bt = sd.Bt_dense()                      # n x m (B~_i^T), original local multiplier order
        br = Bt.T @ Rs[i]                       # B~_i R_i (m x k)
        BR.append(br)
        np.add.at(G, (sd.lambda_map[:, None], off[i] + np.arange(ks[i])[None, :]), br)
        d[sd.lambda_map] += Bt.T @ spla.spsolve(sd.K_reg.tocsc(), fs[i])
        e[off[i]:off[i] + ks[i]] = Rs[i].T @ fs[i]
    return dict(Rs=Rs, ks=ks, off=off[:-1], nc=nc, fs=fs, G=G, d=d, e=e, BR=BR)


def reference_solution(P, D):
    F = np.zeros((P.n_lambda, P.n_lambda))
    for sd, Fi in zip(P.subdomains, oracle.batch_F(P.subdomains)):
        F[np.ix_(sd.lambda_map, sd.lambda_map)] += Fi
    nl, nc = P.n_lambda, D["nc"]
    A = np.block([[F, -D["G"]], [-D["G"].T, np.zeros((nc, nc))]])
    sol = np.linalg.solve(A, np.concatenate([D["d"], -D["e"]]))
    return sol[:nl], sol[nl:], F


def primal_residuals(P, D, lam, alpha):
    """max relative gluing residual ||B u|| / ||u|| and equilibrium residual of u."""
    Bu = np.zeros(P.n_lambda)
    eq = 0.0
    unorm = 0.0
    for i, sd in enumerate(P.subdomains):
        Bt = sd.Bt_dense()
        rhs = D["fs"][i] - Bt @ lam[sd.lambda_map]
        u = spla.spsolve(sd.K_reg.tocsc(), rhs) + D["Rs"][i] @ alpha[D["off"][i]:D["off"][i] + D["ks"][i]]
        Bu[sd.lambda_map] += Bt.T @ u
        K = subdomain_K(P, sd)
        eq = max(eq, np.linalg.norm(K @ u - rhs) / np.linalg.norm(rhs))
        unorm = max(unorm, np.linalg.norm(u))
    return np.linalg.norm(Bu) / unorm, eq
