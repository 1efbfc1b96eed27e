"""Solution stage: PCPG on the FETI dual problem driving sc_apply.

CPU pins (-m "not gpu"): the kernel bases are kernels (K_i R_i = 0), and the dense reference solution
of the dual problem built from the oracle's F_i reproduces the primal FEM solution (gluing B u = 0,
equilibrium K_i u_i = f_i - B~_i^T lambda_i).  GPU (-m gpu): sc_pcpg's lambda and alpha against the
reference, and the same primal residuals from the GPU's lambda / alpha."""
import numpy as np
import pytest

from feti_ref import feti_data, primal_residuals, reference_solution
from synth import config_problem, kernel_basis, subdomain_K


@pytest.mark.parametrize("cfg", ["t2d", "t3e"])
def test_kernel_basis_is_kernel(cfg):
    P = config_problem(cfg)
    for sd in P.subdomains[:3]:
        K = subdomain_K(P, sd)
        R = kernel_basis(P, sd)
        assert np.linalg.norm(K @ R) <= 1e-12 * np.abs(K).max() * np.linalg.norm(R)
        # the regularised inverse is a generalized inverse of K: K K_reg^-1 K = K
        Kd = K.toarray()
        KKK = Kd @ np.linalg.solve(sd.K_reg.toarray(), Kd)
        assert np.linalg.norm(KKK - Kd) <= 1e-9 * np.linalg.norm(Kd)


@pytest.mark.parametrize("cfg", ["cfg1", "t3e"])
def test_reference_dual_solution_is_primal_solution(cfg):
    P = config_problem(cfg)
    D = feti_data(P)
    lam, alpha, _ = reference_solution(P, D)
    glue, eq = primal_residuals(P, D, lam, alpha)
    assert glue <= 1e-9 and eq <= 1e-9
    assert np.linalg.norm(D["G"].T @ lam - D["e"]) <= 1e-9 * np.linalg.norm(D["e"])


def _run_gpu(P, D, **kw):
    import torch
    from paper_2509_21037_b200 import SCPlan
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, **kw)
    Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in P.subdomains]
    plan.assemble(Ls)
    # B~_i R_i column-major (m x k) = a row-major k x m buffer
    coarse = dict(nc=D["nc"], k=D["ks"], off=D["off"],
                  Rt=[torch.from_numpy(np.ascontiguousarray(br.T)).cuda() for br in D["BR"]],
                  GtG_inv=torch.from_numpy(np.linalg.inv(D["G"].T @ D["G"])).cuda())
    d = torch.from_numpy(D["d"]).cuda()
    lam = torch.zeros(P.n_lambda, dtype=torch.float64, device="cuda")
    alpha = torch.zeros(D["nc"], dtype=torch.float64, device="cuda")
    it, rel, hist = plan.pcpg(d, lam, e=D["e"], coarse=coarse, rtol=1e-12, max_it=2000, alpha=alpha, history=2000)
    return lam.cpu().numpy(), alpha.cpu().numpy(), it, rel, hist


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "t2d", "t3d", "t3e"])
def test_pcpg_matches_reference(cfg):
    P = config_problem(cfg)
    D = feti_data(P)
    lam_ref, alpha_ref, F = reference_solution(P, D)
    lam, alpha, it, rel, hist = _run_gpu(P, D)
    assert rel <= 1e-12 and 0 < it < 2000
    assert hist[-1] < hist[0]
    # lambda is unique only up to ker F (the x=0 Dirichlet multipliers and the gluing multiplier of a
    # shared x=0 node are dependent constraints); F lambda, alpha and the primal u are unique
    assert np.linalg.norm(F @ (lam - lam_ref)) <= 1e-8 * np.linalg.norm(F @ lam_ref)
    assert np.linalg.norm(D["G"].T @ lam - D["e"]) <= 1e-9 * np.linalg.norm(D["e"])
    assert np.linalg.norm(alpha - alpha_ref) <= 1e-8 * np.linalg.norm(alpha_ref)
    glue, eq = primal_residuals(P, D, lam, alpha)
    assert glue <= 1e-8 and eq <= 1e-8


@pytest.mark.gpu
def test_pcpg_fp32_mode_and_warp_trsm():
    """PCPG on an FP32-assembled F (precision 32) converges to the FP64 reference within 1e-4."""
    import torch
    from paper_2509_21037_b200 import SCPlan
    P = config_problem("t2d")
    D = feti_data(P)
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, precision=32)
    plan.assemble([torch.from_numpy(np.ascontiguousarray(sd.L_values, dtype=np.float32)).cuda() for sd in P.subdomains])
    coarse = dict(nc=D["nc"], k=D["ks"], off=D["off"],
                  Rt=[torch.from_numpy(np.ascontiguousarray(br.T)).cuda() for br in D["BR"]],
                  GtG_inv=torch.from_numpy(np.linalg.inv(D["G"].T @ D["G"])).cuda())
    lam = torch.zeros(P.n_lambda, dtype=torch.float64, device="cuda")
    it, rel, _ = plan.pcpg(torch.from_numpy(D["d"]).cuda(), lam, e=D["e"], coarse=coarse, rtol=1e-9, max_it=2000)
    assert rel <= 1e-9
    lam_ref, alpha_ref, F = reference_solution(P, D)
    assert np.linalg.norm(F @ (lam.cpu().numpy() - lam_ref)) <= 1e-4 * np.linalg.norm(F @ lam_ref)
