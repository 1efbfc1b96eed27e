"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): plan, assemble (both
TRSM kernels, shared and global strips), explicit and implicit apply, export F; checked against the
oracle so a silent corruption also fails.  Usage: python tools/sanitize_run.py cfg1|t3e|t2d"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2509_21037_b200 import SCPlan  # noqa: E402
from synth import config_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
P = config_problem(cfg)
subs = P.subdomains[:4]
Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in subs]
refs = [oracle.subdomain_F(sd) for sd in subs]
lam = torch.from_numpy(np.random.default_rng(0).standard_normal(P.n_lambda)).cuda()
worst = 0.0
for kw in (dict(trsm_kernel=1, x_strip=1, tile_cols=16), dict(trsm_kernel=1, x_strip=2, tile_cols=16),
           dict(trsm_kernel=2, tile_cols=16), dict(trsm_kernel=2, tile_cols=8)):
    plan = SCPlan(subs, n_lambda=P.n_lambda, **kw)
    plan.assemble(Ls)
    q = torch.zeros_like(lam)
    plan.apply(lam, q)
    plan.prepare_factor(Ls)
    plan.apply_implicit(lam, q)
    torch.cuda.synchronize()
    plan.check()
    for i, F in enumerate(refs):
        worst = max(worst, float(np.linalg.norm(plan.get_F(i) - F) / np.linalg.norm(F)))
    plan.destroy()
print(f"sanitize_run {cfg}: max rel error {worst:.2e}")
assert worst < 1e-10
