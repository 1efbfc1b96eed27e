"""Input-generator checks (CPU): the factor really factors P K_reg P^T, the gluing is consistent,
ND is a permutation, and the configs have the sizes SURVEY.md §8.0 derived."""
import numpy as np
import pytest
import scipy.sparse as sp

from synth import config_problem, make_problem
from synth.mesh import nested_dissection_nodes


@pytest.mark.parametrize("spec", [dict(dim=2, physics="heat", S=2, E=5), dict(dim=3, physics="heat", S=2, E=4),
                                  dict(dim=3, physics="elasticity", S=2, E=3, coef="element")])
def test_factor_reconstruction(spec):
    """||P K P^T - L L^T|| / ||K|| < 1e-12."""
    P = make_problem(**spec)
    for sd in P.subdomains[:3]:
        L = sp.csc_matrix((sd.L_values, sd.L_rowidx, sd.L_colptr), shape=(sd.n, sd.n))
        C = sd.K_reg[sd.perm][:, sd.perm]
        assert sp.linalg.norm(C - L @ L.T) / sp.linalg.norm(C) < 1e-12
        # CSC layout the plan expects: diagonal first, rows ascending
        for c in range(sd.n):
            rows = sd.L_rowidx[sd.L_colptr[c]:sd.L_colptr[c + 1]]
            assert rows[0] == c and np.all(np.diff(rows) > 0)


def test_gluing_consistency():
    """B u = 0 for any continuous field sampled on the global mesh (SPEC problem_gen invariant),
    ignoring the Dirichlet rows (which pin u=0 on x=0)."""
    S, E = 3, 4
    P = make_problem(dim=2, physics="heat", S=S, E=E, dirichlet=False)
    NG = S * E + 1
    rng = np.random.default_rng(0)
    u_glob = rng.standard_normal(NG * NG)
    r = np.zeros(P.n_lambda)
    for sd in P.subdomains:
        sx, sy = sd.id % S, sd.id // S
        loc = np.arange((E + 1) ** 2)
        gx = sx * E + loc % (E + 1)
        gy = sy * E + loc // (E + 1)
        u = u_glob[gx + NG * gy]
        np.add.at(r, sd.lambda_map, sd.Bt_sparse().T @ u)
    assert np.abs(r).max() < 1e-14
    # every gluing multiplier appears in exactly two subdomains with opposite signs
    cnt = np.zeros(P.n_lambda)
    for sd in P.subdomains:
        np.add.at(cnt, sd.lambda_map, 1)
    assert np.all(cnt == 2)


@pytest.mark.parametrize("d,N", [(2, 9), (3, 7), (3, 17)])
def test_nested_dissection_is_permutation(d, N):
    o = nested_dissection_nodes(d, N)
    assert sorted(o.tolist()) == list(range(N ** d))


@pytest.mark.parametrize("cfg,n,nnzL,mmean", [("cfg1", 81, 714, 28), ("cfg2", 4225, 106510, 252),
                                              ("cfg3", 4913, 634564, 1477)])
def test_config_sizes_match_survey(cfg, n, nnzL, mmean):
    P = config_problem(cfg)
    sd = P.subdomains[0]
    assert sd.n == n
    assert sd.L_colptr[-1] == nnzL
    assert abs(np.mean([s.m for s in P.subdomains]) - mmean) < 1.0
