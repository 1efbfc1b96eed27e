import sys, numpy as np, scipy.sparse as sp, torch
sys.path.insert(0, '/root/repo')
from synth import config_problem
from paper_2509_21037_b200 import SCPlan
import oracle
P = config_problem(sys.argv[1])
subs = P.subdomains[:4]
for T, xs, pw in [(16,0,0),(32,0,0),(16,2,0),(32,2,0),(16,0,8),(16,0,64)]:
    plan = SCPlan(subs, n_lambda=P.n_lambda, tile_cols=T, x_strip=xs, panel_cols=pw)
    Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in subs]
    plan.assemble(Ls); torch.cuda.synchronize(); plan.check()
    out = []
    for i, sd in enumerate(subs):
        X, sigma = plan.get_X(i)
        L = sp.csc_matrix((sd.L_values, sd.L_rowidx, sd.L_colptr), shape=(sd.n, sd.n))
        Bt = sd.Bt_dense()[sd.perm][:, sigma]
        R = L @ X - Bt
        res = np.linalg.norm(R) / np.linalg.norm(Bt)
        bad_rows = np.nonzero(np.abs(R).max(axis=1) > 1e-9)[0]
        F = plan.get_F(i); Fo = oracle.subdomain_F(sd)
        out.append((f"{res:.1e}", len(bad_rows), bad_rows[:5].tolist(), f"{np.linalg.norm(F-Fo)/np.linalg.norm(Fo):.1e}"))
    print(T, xs, pw, plan.stats()['panel_cols'], out, flush=True)
