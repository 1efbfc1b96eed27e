"""Print planner statistics for configs (host only): python tools/plan_stats.py cfg2 cfg3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21037_b200 import SCPlan  # noqa: E402
from synth import config_problem  # noqa: E402

for c in sys.argv[1:]:
    P = config_problem(c)
    s = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1).stats()
    print(f"{c}: T={s['tile_cols']} G={s['group_cols']} panels/sub={s['panels'] / s['nsub']:.0f} "
          f"steps/task={s['trsm_steps'] / max(s['trsm_tasks'], 1):.1f} tasks={s['trsm_tasks']} pairs={s['syrk_tasks']} "
          f"execT={s['flops_trsm_executed']:.3g} execS={s['flops_syrk_executed']:.3g} "
          f"useT={s['flops_trsm_useful']:.3g} useS={s['flops_syrk_useful']:.3g} "
          f"PB={s['bytes_panels'] / 1e9:.2f}GB L={s['bytes_L_values'] / 1e9:.2f}GB X={s['bytes_X'] / 1e9:.2f}GB")
