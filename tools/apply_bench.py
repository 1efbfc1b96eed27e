import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from synth import config_problem
from paper_2509_21037_b200 import SCPlan
c = sys.argv[1]
P = config_problem(c)
plan = SCPlan(P.subdomains, n_lambda=P.n_lambda)
Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in P.subdomains]
plan.assemble(Ls); torch.cuda.synchronize()
lam = torch.randn(P.n_lambda, dtype=torch.float64, device='cuda'); q = torch.empty_like(lam)
for _ in range(5): plan.apply(lam, q)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(50): plan.apply(lam, q)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 50
st = plan.stats()
print(c, sys.argv[2] if len(sys.argv) > 2 else '', f"{t:.4f} ms", f"{st['bytes_apply'] / t / 1e6:.0f} GB/s", float(q.sum()))
