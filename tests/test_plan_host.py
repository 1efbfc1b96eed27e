"""Host-only tests of the C ABI (no GPU): the library loads and exports every declared symbol, the
symbolic plan (stepped order, reach strips) is a superset of the brute-force pattern of
X = L^{-1} P B~^T(:, sigma), the work counters reproduce the paper's 3x closed form,
and invalid inputs are rejected with the documented status codes."""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2509_21037_b200 import SCPlan, ScError, SKIP_ENVELOPE, SKIP_EXACT, SKIP_NONE, lib
from paper_2509_21037_b200 import sc as scmod
from synth import config_problem, make_problem
from synth.mesh import Subdomain, custom_problem
from helpers import copy_sd as _copy_sd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sc_b200.h")).read()
    declared = set(re.findall(r"\b(sc_[A-Za-z_]+)\s*\(", hdr))
    L = lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(scmod.EXPORTS)


def _dense_X_pattern(sd):
    """Brute force: structural pattern of L^{-1} P B~^T in exact arithmetic (any non-zero operand
    can make an entry non-zero), by boolean forward substitution."""
    n = sd.n
    Lp, Li = sd.L_colptr, sd.L_rowidx
    iperm = np.empty(n, dtype=np.int64)
    iperm[sd.perm] = np.arange(n)
    pats = []
    for j in range(sd.m):
        nz = np.zeros(n, dtype=bool)
        for p in range(sd.Bt_colptr[j], sd.Bt_colptr[j + 1]):
            nz[iperm[sd.Bt_rowidx[p]]] = True
        for c in range(n):
            if nz[c]:
                nz[Li[Lp[c] + 1:Lp[c + 1]]] = True
        pats.append(np.nonzero(nz)[0])
    return pats


@pytest.mark.parametrize("cfg", ["cfg1", "t3d", "t3e"])
@pytest.mark.parametrize("skip", [SKIP_EXACT, SKIP_ENVELOPE, SKIP_NONE])
def test_strips_cover_structural_pattern(cfg, skip):
    P = config_problem(cfg)
    subs = P.subdomains[:5]
    plan = SCPlan(subs, n_lambda=P.n_lambda, skip=skip, tile_cols=16, device=-1)
    for i, sd in enumerate(subs):
        pats = _dense_X_pattern(sd)
        sigma = plan.sigma(i)
        for a in range(sd.m):
            rows = set(plan.strip_rows(i, a).tolist())
            need = set(pats[sigma[a]].tolist())
            assert need <= rows
            if skip == SKIP_ENVELOPE:
                # the paper's envelope (rows at or below the tile's highest pivot), rounded out to
                # whole factor panels (at most one panel, < 64 rows, above the pivot)
                t0 = (a // 16) * 16
                pmin = min(pats[sigma[b]].min() for b in range(t0, min(t0 + 16, sd.m)))
                assert set(range(pmin, sd.n)) <= rows
                assert min(rows) > pmin - 64 and rows == set(range(min(rows), sd.n))
            if skip == SKIP_NONE:
                assert rows == set(range(sd.n))


def test_stepped_order_pivots_nondecreasing_and_stable():
    P = config_problem("t3e")
    sd = P.subdomains[3]
    plan = SCPlan([sd], n_lambda=P.n_lambda, device=-1)
    sigma = plan.sigma(0)
    iperm = np.empty(sd.n, dtype=np.int64)
    iperm[sd.perm] = np.arange(sd.n)
    piv = np.array([iperm[sd.Bt_rowidx[sd.Bt_colptr[j]:sd.Bt_colptr[j + 1]]].min() for j in range(sd.m)])
    ps = piv[sigma]
    assert np.all(np.diff(ps) >= 0)
    for a in range(sd.m - 1):  # ties keep the original column order
        if ps[a] == ps[a + 1]:
            assert sigma[a] < sigma[a + 1]
    assert sorted(sigma.tolist()) == list(range(sd.m))


def test_stepped_hand_case():
    """column pivots [3,0,2] -> stepped order [1,2,0]."""
    n = 4
    K = sp.identity(n, format="csr") * 2.0
    Bt = np.zeros((n, 3))
    Bt[3, 0] = Bt[0, 1] = Bt[2, 2] = 1.0
    P = custom_problem(K, Bt)
    plan = SCPlan(P.subdomains, n_lambda=3, device=-1)
    assert plan.sigma(0).tolist() == [1, 2, 0]


def _triangular_problem(n, m):
    """Dense lower L (one supernode, etree a chain) and a perfectly triangular B~^T with column
    pivots p_i = floor(i n / m) (reading of SURVEY §8.3 item 12)."""
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(np.arange(n, 0, -1))
    rowidx = np.concatenate([np.arange(c, n, dtype=np.int32) for c in range(n)])
    piv = (np.arange(m) * n) // m
    sd = Subdomain(0, n, 1.0, np.arange(n, dtype=np.int32), colptr, rowidx, np.arange(m + 1, dtype=np.int32),
                   piv.astype(np.int32), np.ones(m), np.arange(m, dtype=np.int64))
    return sd


def test_theoretical_speedup_three():
    """dense TRSM and SYRK on a perfectly triangular RHS do 3x the work of the stepped
    version (pyramid in a prism)."""
    n = m = 2048
    plan = SCPlan([_triangular_problem(n, m)], n_lambda=m, device=-1)
    s = plan.stats()
    r_trsm = s["flops_trsm_dense"] / s["flops_trsm_envelope"]
    r_syrk = s["flops_syrk_dense"] / s["flops_syrk_envelope"]
    assert abs(r_trsm - 3.0) < 0.01 and abs(r_syrk - 3.0) < 0.01
    # single-supernode dense factor: exact reach == envelope
    assert s["flops_trsm_useful"] == s["flops_trsm_envelope"]
    assert s["flops_syrk_useful"] == s["flops_syrk_envelope"]


def test_work_counters_match_survey_cfg2_cfg3():
    for cfg, useful, env in [("cfg2", 1.09e10, 1.20e11), ("cfg3", 5.97e11, 2.54e12)]:
        P = config_problem(cfg)
        s = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1).stats()
        u = s["flops_trsm_useful"] + s["flops_syrk_useful"]
        e = s["flops_trsm_envelope"] + s["flops_syrk_envelope"]
        assert abs(u / useful - 1) < 0.02 and abs(e / env - 1) < 0.02
        # monotone: useful <= envelope <= dense
        assert s["flops_trsm_useful"] <= s["flops_trsm_envelope"] <= s["flops_trsm_dense"]
        assert s["flops_syrk_useful"] <= s["flops_syrk_envelope"] <= s["flops_syrk_dense"]


def test_pattern_classes_dedup():
    P = config_problem("cfg1")
    s = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1).stats()
    assert s["n_classes"] == 9  # 3 x 3 boundary classes of a 4x4 decomposition




def test_invalid_inputs_rejected():
    P = config_problem("cfg1")
    sd = P.subdomains[0]
    # diagonal not first
    ri = sd.L_rowidx.copy()
    ri[sd.L_colptr[3]], ri[sd.L_colptr[3] + 1] = ri[sd.L_colptr[3] + 1], ri[sd.L_colptr[3]]
    with pytest.raises(ScError) as e:
        SCPlan([_copy_sd(sd, L_rowidx=ri)], n_lambda=P.n_lambda, device=-1)
    assert e.value.status == scmod.SC_ERR_PATTERN
    # perm not a bijection
    pm = sd.perm.copy()
    pm[0] = pm[1]
    with pytest.raises(ScError) as e:
        SCPlan([_copy_sd(sd, perm=pm)], n_lambda=P.n_lambda, device=-1)
    assert e.value.status == scmod.SC_ERR_PATTERN
    # B row out of range
    br = sd.Bt_rowidx.copy()
    br[0] = sd.n
    with pytest.raises(ScError) as e:
        SCPlan([_copy_sd(sd, Bt_rowidx=br)], n_lambda=P.n_lambda, device=-1)
    assert e.value.status == scmod.SC_ERR_PATTERN
    # lambda_map out of range
    with pytest.raises(ScError) as e:
        SCPlan([sd], n_lambda=1, device=-1)
    assert e.value.status == scmod.SC_ERR_INVALID_ARG
    # bad tile size
    with pytest.raises(ScError) as e:
        SCPlan([sd], n_lambda=P.n_lambda, tile_cols=48, device=-1)
    assert e.value.status == scmod.SC_ERR_INVALID_ARG
    # bad strip mode
    with pytest.raises(ScError) as e:
        SCPlan([sd], n_lambda=P.n_lambda, x_strip=3, device=-1)
    assert e.value.status == scmod.SC_ERR_INVALID_ARG


def test_global_strip_plan_same_reach_and_work():
    """The global-strip variant (tiles solved in place in the SYRK group strip) visits the same
    panels as the shared-memory variant: identical strip rows, executed and useful work."""
    P = config_problem("t3e")
    subs = P.subdomains[:6]
    a = SCPlan(subs, n_lambda=P.n_lambda, tile_cols=16, x_strip=scmod.STRIP_SHARED, device=-1)
    b = SCPlan(subs, n_lambda=P.n_lambda, tile_cols=16, x_strip=scmod.STRIP_GLOBAL, device=-1,
               trsm_kernel=scmod.TRSM_CTA)
    sa, sb = a.stats(), b.stats()
    assert sa["x_strip"] == scmod.STRIP_SHARED and sb["x_strip"] == scmod.STRIP_GLOBAL
    for k in ("flops_trsm_useful", "flops_syrk_useful", "flops_trsm_executed", "flops_syrk_executed", "bytes_X",
              "trsm_steps", "syrk_tasks"):
        assert sa[k] == sb[k], k
    for i, sd in enumerate(subs):
        for col in range(0, sd.m, 16):
            assert np.array_equal(a.strip_rows(i, col), b.strip_rows(i, col))


def test_not_fill_closed_pattern_rejected():
    """Arrow matrix factor with its fill dropped: not a Cholesky pattern -> SC_ERR_PATTERN."""
    # columns: 0 -> rows {0, 2, 3}; 1 -> {1, 2}; 2 -> {2}; 3 -> {3}: parent(0)=2 but row 3 not in struct(2)
    colptr = np.array([0, 3, 5, 6, 7], dtype=np.int64)
    rowidx = np.array([0, 2, 3, 1, 2, 2, 3], dtype=np.int32)
    sd = Subdomain(0, 4, 1.0, np.arange(4, dtype=np.int32), colptr, rowidx, np.array([0, 1], dtype=np.int32),
                   np.array([0], dtype=np.int32), np.array([1.0]), np.array([0], dtype=np.int64))
    with pytest.raises(ScError) as e:
        SCPlan([sd], n_lambda=1, device=-1)
    assert e.value.status == scmod.SC_ERR_PATTERN


def test_host_only_plan_refuses_device_calls():
    P = config_problem("cfg1")
    plan = SCPlan(P.subdomains[:2], n_lambda=P.n_lambda, device=-1)
    with pytest.raises(ScError) as e:
        plan.get_F(0)
    assert e.value.status == scmod.SC_ERR_STATE


def test_empty_subdomain_and_empty_columns():
    P = config_problem("cfg1")
    sd = P.subdomains[0]
    empty = _copy_sd(sd, m=0, Bt_colptr=np.zeros(1, dtype=np.int32), Bt_rowidx=np.zeros(0, dtype=np.int32),
                     Bt_values=np.zeros(0), lambda_map=np.zeros(0, dtype=np.int64))
    # a column with no non-zero sorts last (sentinel pivot n)
    bc = np.concatenate([[0], np.cumsum([1, 0, 1])]).astype(np.int32)
    holes = _copy_sd(sd, m=3, Bt_colptr=bc, Bt_rowidx=sd.Bt_rowidx[:2].copy(), Bt_values=np.array([1.0, -1.0]),
                     lambda_map=np.arange(3, dtype=np.int64))
    plan = SCPlan([empty, holes], n_lambda=P.n_lambda, device=-1)
    assert plan.sigma(1)[-1] == 1
    assert plan.stats()["sum_m"] == 3


def test_auto_tile_and_strip_selection_defaults():
    """The planner's measured defaults: 2D cfg2 -> warp TRSM at T=16 in the global
    strips, 32-wide panels; 3D (cfg3, cfg4) -> CTA TRSM at T=16 global strips at two CTAs per SM,
    64-wide panels."""
    from synth import make_problem
    cases = [(dict(dim=2, physics="heat", S=32, E=64), 16, scmod.STRIP_GLOBAL, "none", 32, scmod.TRSM_WARP),
             (dict(dim=3, physics="heat", S=8, E=16), 16, scmod.STRIP_GLOBAL, "none", 64, scmod.TRSM_CTA),
             (dict(dim=3, physics="elasticity", S=8, E=12), 16, scmod.STRIP_GLOBAL, "none", 64, scmod.TRSM_CTA)]
    for spec, T, strip, two_cta, pw, kern in cases:
        P = make_problem(subdomains=[0, 5, spec["S"] ** spec["dim"] // 2], **spec)
        st = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1).stats()
        assert st["tile_cols"] == T and st["x_strip"] == strip and st["panel_cols"] == pw, (spec, st["tile_cols"])
        assert st["trsm_kernel"] == kern
        if two_cta == "all":
            assert st["trsm_tasks_2cta"] == st["trsm_tasks"] > 0
        else:
            assert st["trsm_tasks_2cta"] == 0
