"""Seeded synthetic FETI inputs (input generator only; holds none of the method's arithmetic).

This module builds what the paper's preprocessing receives (§3: "The input for
the algorithm is the matrix B~_i^T together with the factor L_i"): per subdomain the regularised
stiffness K_reg (for the oracle), its fill-reducing permutation and sparse Cholesky factor L (for
the GPU path), the signed-Boolean gluing B~_i^T and the local->global multiplier map.

It is the only code shared by the oracle side and the CUDA side (it is test/bench input
generation).  Recipe: structured Q1 meshes on the unit square/cube, S subdomains
per axis of E elements each; heat (1 DOF/node) or linear elasticity (3 DOF/node, nu=0.3);
coefficient per subdomain kappa_i ~ U[1,10) from (seed, i) (optionally per element); fixing-node
regularisation rho = mean(diag K); non-redundant gluing plus Dirichlet on x=0 through B;
geometric nested-dissection ordering.
"""
from .mesh import (  # noqa: F401
    Problem,
    Subdomain,
    CONFIGS,
    make_problem,
    config_problem,
    chain_1d_problem,
    custom_problem,
    kernel_basis,
    subdomain_K,
)
