import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from synth import make_problem
from paper_2509_21037_b200 import SCPlan
import oracle
P = make_problem(dim=3, physics="elasticity", S=8, E=12, subdomains=[0, 73])
T = int(sys.argv[1]) if len(sys.argv) > 1 else 32
xs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, tile_cols=T, x_strip=xs)
print(plan.stats()['tile_cols'], plan.stats()['x_strip'], flush=True)
Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in P.subdomains]
plan.assemble(Ls); torch.cuda.synchronize(); plan.check()
sd = P.subdomains[1]
cols = [0, 5, sd.m - 1]
F = plan.get_F(1)[:, cols]
Fo = oracle.subdomain_F(sd, cols)
print("err", np.linalg.norm(F - Fo) / np.linalg.norm(Fo))
