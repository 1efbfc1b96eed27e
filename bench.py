#!/usr/bin/env python
"""Benchmark of the batched explicit Schur-complement assembly (arXiv 2509.21037 hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One step = one sc_assemble_batch over the config's whole batch of subdomains (X init + stepped
supernodal TRSM + block-sparse SYRK), with the L values resident in HBM.  Multi-GPU (torchrun):
one process per GPU; by default the config's ONE batch is partitioned over the ranks by LPT on the
planner's per-subdomain cost (strong scaling, BASELINE cfg3 "512 subdomains sharded
over 1/2/4/8"); `--weak` gives every rank its own replica batch instead.  No collective
on the assembly path; time = max over ranks of the CUDA-event time.  `--impl reference` times the CPU oracle (oracle/) on the host cores
on a bounded sample of the same workload (rank 0 only).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_A100_MS = {  # PAPER.md Fig. 8 "sep", optimized GPU, per subdomain (context only, A100)
    "cfg1": 0.0470,  # 2D n=81
    "cfg2": 0.5441,  # 2D n=4,225
    "cfg3": 2.008,   # 3D n=4,913
}
METRIC = "SC assembly subdomains/s + FP64 GFLOP/s at 1/2/4/8 B200; amortization iters"
CFG_DESC = {
    "cfg1": "2D heat 4x4=16 subdomains of 8x8 Q1 (81 DOF)",
    "cfg2": "2D heat 1024 subdomains of 64x64 Q1 (4225 DOF)",
    "cfg3": "3D heat 512 subdomains of 16^3 Q1 hex (4913 DOF)",
    "cfg4": "3D elasticity 512 subdomains of 12^3 Q1 hex (6591 DOF)",
    "cfg5": "3D elasticity 64 subdomains of 24^3 Q1 hex (46875 DOF)",
}


def load_peaks():
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peaks.update(json.load(open(p)))
    # FP64 DMMA peak measured on this pool's B200 by tools/fp64_peak.cu (profiles/fp64_peak_r01.txt)
    peaks.setdefault("fp64_tflops", 37.108)
    peaks.setdefault("fp64_tflops_source", "measured: tools/fp64_peak.cu DMMA.8x8x4 loop, profiles/fp64_peak_r01.txt")
    if "hbm_gbs" not in peaks:
        peaks["hbm_gbs"] = 6650.0
        peaks["hbm_source"] = "fallback (B200_PROFILING.md)"
    else:
        peaks.setdefault("hbm_source", "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)")
    return peaks


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled from
    a background thread every ~2 ms (the timed region can be tens of ms), plus one sample at entry
    and one at exit.  Falls back to nvidia-smi if NVML is unavailable."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = None
        self._thr = None

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.rows.append((sm, rs))

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._stop = threading.Event()

            def loop():
                while not self._stop.wait(0.002):
                    try:
                        self._sample()
                    except Exception:
                        break
            self._thr = threading.Thread(target=loop, daemon=True)
            self._thr.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *a):
        if self._thr:
            self._stop.set()
            self._thr.join(timeout=2)
        if getattr(self, "h", None) is not None:
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        import pynvml
        names = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                 "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                 "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                 "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({nm for _, rs in self.rows for nm, bit in names.items() if rs & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, ~2 ms polling during the timed region"}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(problem, budget_s: float, threads: int):
    """Oracle (as it stands) over subdomains of the workload, one subdomain per host thread, until
    `budget_s` elapses; returns (subdomains/s, subdomains done, wall seconds)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    subs = problem.subdomains
    done, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        while True:
            batch = [subs[(done + k) % len(subs)] for k in range(threads)]
            list(ex.map(oracle.subdomain_F, batch))
            done += len(batch)
            if time.perf_counter() - t0 >= budget_s:
                break
    wall = time.perf_counter() - t0
    return done / wall, done, wall


def run_reference(args, world, rank):
    if rank != 0:
        return
    from synth import config_problem
    P = config_problem(args.config)
    threads = len(os.sched_getaffinity(0))
    per_step = []
    total_done, total_wall = 0, 0.0
    for k in range(args.warmup + args.steps):
        v, done, wall = cpu_oracle_sample(P, args.ref_budget, threads)
        if k >= args.warmup:
            per_step.append(wall / done)
            total_done += done
            total_wall += wall
    value = total_done / total_wall
    useful = None
    sample = (f"{args.steps} steps x >= {args.ref_budget:.0f}s of oracle work each, one subdomain per thread "
              f"({total_done} subdomains of {args.config}), extrapolated as subdomains/s")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "subdomains/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * len(P.subdomains) / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CFG_DESC[args.config], "subdomains": len(P.subdomains)},
            "cpu_baseline": {"value": value, "unit": "subdomains/s", "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": "subdomains/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def setup_problem(args, cfg, world, rank):
    """This rank's subdomains: its LPT share of the config's batch (default) or a replica (--weak)."""
    from paper_2509_21037_b200 import SCPlan
    from synth import config_problem
    from synth.mesh import CONFIGS, make_problem
    if args.weak or world == 1:
        if args.perturbed:  # one fill-reducing ordering (L pattern) per subdomain: plan-time / memory stress
            return make_problem(name=cfg, perturbed=True, seed=rank if args.weak else 0, **CONFIGS[cfg]), None
        return config_problem(cfg, seed=rank if args.weak else 0), None
    from paper_2509_21037_b200.shard import imbalance, lpt_partition
    Pall = make_problem(name=cfg, perturbed=True, **CONFIGS[cfg]) if args.perturbed else config_problem(cfg)
    costs = SCPlan(Pall.subdomains, n_lambda=Pall.n_lambda, device=-1).subdomain_costs()
    parts = lpt_partition(costs, world)
    P = make_problem(name=cfg, subdomains=parts[rank], perturbed=args.perturbed, **CONFIGS[cfg])
    info = {"nsub_total": len(Pall.subdomains), "imbalance": imbalance(costs, parts),
            "partition": "LPT on the planner's executed-flop cost", "nsub_per_rank": [len(p) for p in parts]}
    return P, info


def time_assembly(plan, Ls, steps, warmup, world, clock_index=None):
    """W untimed + K timed sc_assemble_batch calls; CUDA events on the launching stream (per phase
    inside the call); barrier + synchronize on both sides; returns (ms_total, phase ms, clocks)."""
    import torch
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    Lp = plan.pointer_array(Ls)  # the C pointer array, built once (not re-marshalled per call)
    for _ in range(warmup):
        plan.assemble(Lp)
    torch.cuda.synchronize()
    plan.check()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    for row in evs:  # torch creates the CUDA event lazily on first record
        for e in row:
            e.record(stream)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(clock_index if clock_index is not None else torch.cuda.current_device()) as clk:
        start.record(stream)
        for k in range(steps):
            plan.set_timing_events(evs[k])
            plan.assemble(Lp)
        stop.record(stream)
        torch.cuda.synchronize()
    plan.set_timing_events(None)
    if world > 1:
        dist.barrier()
    plan.check()
    phases = {"prep": sum(e[0].elapsed_time(e[1]) for e in evs) / steps,
              "trsm": sum(e[1].elapsed_time(e[2]) for e in evs) / steps,
              "syrk": sum(e[2].elapsed_time(e[3]) for e in evs) / steps}
    return start.elapsed_time(stop), phases, clk.summary()


def time_factor(plan, P, steps, warmup, peaks):
    """Device numeric factorization: sc_factorize_batch (device K -> device L) timed with
    CUDA events over `steps` calls, and the device-resident preprocessing factorize + assemble.
    Returns (summary dict, device K tensors, device L tensors)."""
    import torch
    t0 = time.perf_counter()
    plan.factor_attach([sd.K_lower()[:2] for sd in P.subdomains])
    t_sym = time.perf_counter() - t0
    st = plan.stats()
    Kd = [torch.from_numpy(sd.K_lower()[2]).cuda() for sd in P.subdomains]
    Lo = [torch.empty(int(sd.L_colptr[-1]), dtype=torch.float64, device="cuda") for sd in P.subdomains]
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        plan.factorize(Kd, Lo)
    torch.cuda.synchronize()
    plan.check()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(stream)
    for _ in range(steps):
        plan.factorize(Kd, Lo)
    e1.record(stream)
    for _ in range(steps):
        plan.factorize(Kd, Lo)
        plan.assemble(Lo)
    e2.record(stream)
    torch.cuda.synchronize()
    plan.check()
    ms_f = e0.elapsed_time(e1) / steps
    ms_fa = e1.elapsed_time(e2) / steps
    nsub = len(P.subdomains)
    worst = max(float((Lo[i] - torch.from_numpy(P.subdomains[i].L_values).cuda()).abs().max()) /
                float(np.abs(P.subdomains[i].L_values).max()) for i in (0, nsub // 2, nsub - 1))
    out = {"ms": ms_f, "subdomains_per_s": nsub / (ms_f / 1e3),
           "gflops_useful": st["flops_factor_useful"] / (ms_f / 1e3) / 1e9,
           "fp64_frac_useful": st["flops_factor_useful"] / (ms_f / 1e3) / 1e12 / peaks["fp64_tflops"],
           "flops_useful": st["flops_factor_useful"], "flops_executed": st["flops_factor_executed"],
           "bytes_K": st["bytes_K_values"], "bytes_L": st["bytes_L_values"], "tasks": st["factor_tasks"],
           "max_level": st["factor_max_level"], "symbolic_s": t_sym,
           "preprocessing_ms": ms_fa, "preprocessing_subdomains_per_s": nsub / (ms_fa / 1e3),
           "L_vs_host_factor_max_rel_diff": worst,
           "kernel": "factor_kernel (left-looking supernodal, warp per 32-row frame, DMMA updates)",
           "note": "preprocessing = sc_factorize_batch + sc_assemble_batch (P:326-328 two-stage factorization; "
                   "P:2563-2570 factorization share)"}
    return out, Kd, Lo


def roofline_for(st, phases, ms_step, peaks, cfg):
    """Dominant kernel of the step vs the roof its algorithmic intensity selects:
       prep: bytes = L values read once;
       trsm: flops = useful (etree-exact) TRSM flops, bytes = L values read once + X tile-exact
             written once (sc_stats.bytes_X_reach);
       syrk: flops = useful SYRK flops, bytes = X strips read once + F lower written once."""
    dom = max(phases, key=phases.get)
    dom_ms = phases[dom]
    prof_traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg}.json")
    if os.path.exists(tp):
        prof_traffic = json.load(open(tp)).get(dom)
    warp = st.get("trsm_kernel") == 2
    kernel_names = {"prep": "prep_panel_kernel + prep_small_kernel",
                    "trsm": (f"trsm_warp_kernel<{st['tile_cols'] // 8}>" if warp else f"trsm_smem_kernel<{st['tile_cols']}>"),
                    "syrk": ("syrk_warp16_kernel" if st["group_cols"] == 16 else f"syrk_pair_kernel<{st['group_cols']}>")}
    alg = {"prep": (0.0, st["bytes_L_values"]),
           "trsm": (st["flops_trsm_useful"], st["bytes_L_values"] + st["bytes_X_reach"]),
           "syrk": (st["flops_syrk_useful"], st["bytes_X"] + st["bytes_F_lower"])}
    flops, nbytes = alg[dom]
    ridge = peaks["fp64_tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    intensity = flops / nbytes if nbytes else float("inf")
    if intensity < ridge:
        achieved = nbytes / (dom_ms / 1e3) / 1e9
        r = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
             "frac": achieved / peaks["hbm_gbs"], "peak_source": peaks.get("hbm_source", "MEASURED_PEAKS.json hbm_gbs")}
    else:
        achieved = flops / (dom_ms / 1e3) / 1e12
        r = {"bound": "tensor", "achieved": achieved, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
             "frac": achieved / peaks["fp64_tflops"], "dtype": "f64 (DMMA m8n8k4)",
             "peak_source": peaks["fp64_tflops_source"]}
    r.update({"algorithmic": {"prep": "L values read once (8 B/nnz(L))",
                              "trsm": "useful TRSM flops; L values read once + X tile-exact written once",
                              "syrk": "useful SYRK flops; X strips read once + F lower written once"}[dom],
              "algorithmic_flops": flops, "algorithmic_bytes": nbytes, "intensity_flop_per_byte": intensity,
              "ridge_flop_per_byte": ridge, "traffic": prof_traffic, "kernel": kernel_names[dom],
              "share_of_step": dom_ms / ms_step, "launch_ms": dom_ms})
    return r


def per_config_lines(args, peaks):
    """Extra configs timed in the same run (N=1): phase times, throughput and roofline of each, so
    the FP64-bound 3D evidence is measured on the driver's box too."""
    import torch
    from paper_2509_21037_b200 import SCPlan
    from synth import config_problem
    out = {}
    for cfg in [c for c in args.per_config.split(",") if c in CFG_DESC and c != args.config]:
        P = config_problem(cfg)
        t0 = time.perf_counter()
        plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=torch.cuda.current_device())
        t_plan = time.perf_counter() - t0
        st = plan.stats()
        Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in P.subdomains]
        steps = max(2, min(args.steps, 5))
        ms_total, phases, clocks = time_assembly(plan, Ls, steps, 3, 1)
        ms_step = ms_total / steps
        useful = st["flops_trsm_useful"] + st["flops_syrk_useful"]
        fac, Kd, Lo = time_factor(plan, P, steps, 2, peaks)
        del Kd, Lo
        out[cfg] = {"workload": CFG_DESC[cfg], "subdomains": len(P.subdomains), "steps": steps, "warmup": 3,
                    "value": len(P.subdomains) / (ms_step / 1e3), "unit": "subdomains/s", "ms_per_step": ms_step,
                    "phase_ms": phases, "gflops_useful": useful / (ms_step / 1e3) / 1e9,
                    "fp64_frac_useful": useful / (ms_step / 1e3) / 1e12 / peaks["fp64_tflops"],
                    "roofline": roofline_for(st, phases, ms_step, peaks, cfg), "clocks": clocks, "plan_s": t_plan,
                    "tile_cols": st["tile_cols"], "trsm_kernel": {1: "cta", 2: "warp"}.get(st["trsm_kernel"]),
                    "factor": fac}
        del Ls, plan
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=list(CFG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip", default="exact", choices=["none", "envelope", "exact"])
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--panel", type=int, default=0)
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank assembles its own replica batch of the config (default: the "
                         "config's one batch is LPT-partitioned over the ranks by the planner's cost)")
    ap.add_argument("--shard", action="store_true", help="(default; kept for compatibility)")
    ap.add_argument("--strip", default="auto", choices=["auto", "shared", "global"],
                    help="where TRSM tiles keep their X strip (sc_options.x_strip)")
    ap.add_argument("--trsm", default="auto", choices=["auto", "cta", "warp"], help="sc_options.trsm_kernel")
    ap.add_argument("--syrk", default="output", choices=["output", "input"],
                    help="SYRK splitting (P:523-540): output (default) or input (f3 ablation, SC_SYRK_SPLIT=input)")
    ap.add_argument("--per-config", default="cfg3,cfg4",
                    help="extra configs timed in the same run (N=1 only), reported under per_config")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=8.0, help="seconds of oracle work per reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-amortization", action="store_true")
    ap.add_argument("--no-factor", action="store_true", help="skip the device factorization (f4) timing / K-fed e2e")
    ap.add_argument("--perturbed", action="store_true",
                    help="a distinct fill-reducing ordering (L pattern) per subdomain: every subdomain its own plan "
                         "class (plan time / plan memory at the scale of a graph-partitioned mesh)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2509_21037_b200 import SCPlan

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks = load_peaks()

    P, shard_info = setup_problem(args, args.config, world, rank)
    if args.syrk == "input":
        os.environ["SC_SYRK_SPLIT"] = "input"
    import psutil
    rss0 = psutil.Process().memory_info().rss
    t_plan0 = time.perf_counter()
    skip = {"none": 0, "envelope": 1, "exact": 2}[args.skip]
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, skip=skip, tile_cols=args.tile, panel_cols=args.panel,
                  device=local, x_strip={"auto": 0, "shared": 1, "global": 2}[args.strip],
                  trsm_kernel={"auto": 0, "cta": 1, "warp": 2}[args.trsm])
    t_plan = time.perf_counter() - t_plan0
    plan_rss_mb = (psutil.Process().memory_info().rss - rss0) / 1e6
    st = plan.stats()
    Ls = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).cuda() for sd in P.subdomains]
    nsub = len(P.subdomains)
    stream = torch.cuda.current_stream()
    useful = st["flops_trsm_useful"] + st["flops_syrk_useful"]

    ms_total, phases, clocks = time_assembly(plan, Ls, args.steps, args.warmup, world, local)
    t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
    per_rank_ms = [ms_total / args.steps]
    if world > 1:
        allt = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank_ms = [float(x.item()) / args.steps for x in allt]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = t.item() / args.steps
    nsub_job = shard_info["nsub_total"] if shard_info else world * nsub
    # job-wide flops: summed over ranks (each rank's batch differs when sharded)
    fl = torch.tensor([useful, st["flops_trsm_executed"] + st["flops_syrk_executed"]], dtype=torch.float64,
                      device="cuda")
    if world > 1:
        dist.all_reduce(fl)
    useful_job, executed_job = float(fl[0]), float(fl[1])
    value = nsub_job / (ms_step / 1e3)

    # device numeric factorization (f4) and the host-fed end-to-end paths through the public API:
    #   e2e        pinned K values (lower triangle) -> H2D inside sc_factorize_assemble_host -> device
    #              factorization -> assembly -> one explicit apply (NCCL all-reduce for N > 1) -> D2H of q
    #   e2e_from_L pinned L values -> H2D inside sc_assemble_batch_host -> assembly -> apply -> D2H of q
    factor = None
    if not args.no_factor:
        factor, Kd, Lo = time_factor(plan, P, args.steps, args.warmup, peaks)
        del Kd, Lo
    lam_h = torch.from_numpy(np.random.default_rng(0).standard_normal(P.n_lambda)).pin_memory()
    lam_d = torch.empty(P.n_lambda, dtype=torch.float64, device="cuda")
    q_d = torch.empty_like(lam_d)
    q_h = torch.empty(P.n_lambda, dtype=torch.float64).pin_memory()

    def e2e_run(step_fn, h2d_inputs, includes):
        for _ in range(args.warmup):
            step_fn()
            lam_d.copy_(lam_h, non_blocking=True)
            plan.apply_global(lam_d, q_d)
            q_h.copy_(q_d, non_blocking=True)
        torch.cuda.synchronize()
        plan.check()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step_fn()
            lam_d.copy_(lam_h, non_blocking=True)
            plan.apply_global(lam_d, q_d)
            q_h.copy_(q_d, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return {"value": nsub_job / (te.item() / 1e3), "unit": "subdomains/s", "ms_per_step": te.item(),
                "h2d_bytes_per_step": int(h2d_inputs + 8 * P.n_lambda), "d2h_bytes_per_step": 8 * P.n_lambda,
                "includes": includes}

    e2e = e2e_L = None
    if not args.no_e2e:
        hostL = [torch.from_numpy(np.ascontiguousarray(sd.L_values)).pin_memory() for sd in P.subdomains]
        hostLp = plan.pointer_array(hostL)
        e2e_L = e2e_run(lambda: plan.assemble_host(hostLp), sum(8 * sd.L_values.size for sd in P.subdomains),
                        "pinned H2D of this rank's L values + assemble + 1 sc_apply (+NCCL all-reduce) + D2H of q")
        del hostL
        if factor is not None:
            hostK = [torch.from_numpy(sd.K_lower()[2]).pin_memory() for sd in P.subdomains]
            hostKp = (ctypes.c_void_p * max(len(hostK), 1))(*[k.data_ptr() for k in hostK])
            e2e = e2e_run(lambda: plan.factorize_assemble_host(hostKp), sum(8 * k.numel() for k in hostK),
                          "pinned H2D of this rank's K values (lower triangle) + device numeric factorization + "
                          "assemble + 1 sc_apply (+NCCL all-reduce) + D2H of q (sc_factorize_assemble_host)")
            del hostK
        else:
            e2e = e2e_L

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    roofline = roofline_for(st, phases, ms_step * world / world, peaks, args.config)
    # amortization point: explicit GPU (assembly + apply per
    # iteration) vs implicit CPU apply per iteration on the host cores; the factorization is common
    # to both and cancels.  k* = smallest k with t_asm + k t_expl < k t_impl.
    amort = None
    if not args.no_amortization and world == 1:
        lam_d = torch.from_numpy(np.random.default_rng(7).standard_normal(P.n_lambda)).cuda()
        q_d = torch.empty_like(lam_d)
        for _ in range(3):
            plan.apply(lam_d, q_d)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        torch.cuda.synchronize()
        a0.record(stream)
        for _ in range(reps):
            plan.apply(lam_d, q_d)
        a1.record(stream)
        torch.cuda.synchronize()
        t_expl = a0.elapsed_time(a1) / reps
        # GPU implicit apply (two substitutions per subdomain with the staged factor, no F);
        # its up-front cost is the factor staging (sc_prepare_factor), timed here
        for _ in range(2):
            plan.prepare_factor(Ls)
        torch.cuda.synchronize()
        a0.record(stream)
        plan.prepare_factor(Ls)
        a1.record(stream)
        torch.cuda.synchronize()
        t_stage = a0.elapsed_time(a1)
        for _ in range(3):
            plan.apply_implicit(lam_d, q_d)
        torch.cuda.synchronize()
        a0.record(stream)
        for _ in range(reps):
            plan.apply_implicit(lam_d, q_d)
        a1.record(stream)
        torch.cuda.synchronize()
        t_impl_gpu = a0.elapsed_time(a1) / reps
        q_impl_gpu = q_d.cpu().numpy()
        plan.apply(lam_d, q_d)
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from implicit_cpu import ImplicitCPU
        ic = ImplicitCPU(P)
        t_impl = 1e3 * ic.time(reps=5, warmup=1)
        q_impl = ic.apply(lam_d.cpu().numpy())
        agree = float(np.linalg.norm(q_d.cpu().numpy() - q_impl) / np.linalg.norm(q_impl))

        def kstar(t_asm, t_imp, t_up=0.0):
            d = t_imp - t_expl
            return int(max(t_asm - t_up, 0.0) // d) + 1 if d > 0 else None

        amort = {"iters": kstar(ms_step, t_impl), "iters_e2e": kstar(e2e_L["ms_per_step"], t_impl) if e2e_L else None,
                 "iters_vs_gpu_implicit": kstar(ms_step, t_impl_gpu, t_stage), "t_apply_implicit_gpu_ms": t_impl_gpu,
                 "t_factor_staging_gpu_ms": t_stage,
                 "implicit_gpu_vs_explicit_rel_diff": float(np.linalg.norm(q_impl_gpu - q_d.cpu().numpy()) /
                                                            np.linalg.norm(q_d.cpu().numpy())),
                 "t_assembly_ms": ms_step, "t_apply_explicit_gpu_ms": t_expl, "t_apply_implicit_cpu_ms": t_impl,
                 "cpu_threads": ic.used_threads, "explicit_vs_implicit_rel_diff": agree,
                 "paper": "~10 iterations (A100 + 16 EPYC cores, P:56, P:2919)"}
    cpu = None
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        v, done, wall = cpu_oracle_sample(P, args.cpu_budget, threads)
        cpu = {"value": v, "unit": "subdomains/s", "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{done} subdomains of {args.config} ({wall:.1f}s, one subdomain per host thread)"}
    per_config = per_config_lines(args, peaks) if world == 1 and args.per_config else None
    line = {
        "metric": METRIC, "value": value, "unit": "subdomains/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if (args.weak and world > 1) else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CFG_DESC[args.config], "name": args.config, "subdomains_per_gpu": nsub,
                   "skip": args.skip, "tile_cols": st["tile_cols"], "panel_cols": st["panel_cols"],
                   "trsm_kernel": {1: "cta", 2: "warp"}.get(st["trsm_kernel"]),
                   "x_strip": {1: "shared", 2: "global"}.get(st["x_strip"], "?"),
                   "trsm_tasks_2cta": st["trsm_tasks_2cta"], "syrk_split": args.syrk,
                   "parallelism": (f"replica batch per rank x{world}" if (args.weak and world > 1) else
                                   f"one batch LPT-sharded over {world} rank(s), no collective in assembly"),
                   "shard": shard_info, "nccl_ranks": world, "per_rank_ms": per_rank_ms,
                   "rank_imbalance_measured": max(per_rank_ms) / (sum(per_rank_ms) / len(per_rank_ms)),
                   "l2": f"inputs larger than L2: L values {st['bytes_L_values'] / 1e9:.2f} GB, "
                         f"X {st['bytes_X'] / 1e9:.2f} GB, F lower tiles "
                         f"{8 * 4096 * sum(((m + 63) // 64) * ((m + 63) // 64 + 1) // 2 for m in plan.m) / 1e9:.2f} GB per GPU"},
        "gflops_useful": useful_job / (ms_step / 1e3) / 1e9,
        "gflops_executed": executed_job / (ms_step / 1e3) / 1e9,
        "fp64_frac_useful": useful_job / world / (ms_step / 1e3) / 1e12 / peaks["fp64_tflops"],
        "phase_ms": phases,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_from_L": e2e_L, "factor": factor,
        "amortization": amort,
        "gpu_launches": args.steps * plan.launches_per_assemble,
        "clocks": clocks, "plan_s": t_plan, "plan_host_rss_mb": plan_rss_mb, "n_classes": st["n_classes"],
        "patterns": "perturbed: one ordering per subdomain" if args.perturbed else "one per boundary class",
        "per_config": per_config,
        "paper_context": {"a100_sep_opt_ms_per_subdomain": PAPER_A100_MS.get(args.config),
                          "note": "PAPER.md Fig. 8, A100, triangles/tets; context only"},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
