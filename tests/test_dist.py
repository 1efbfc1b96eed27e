"""Multi-process (world size 2, gloo, CPU) tests of the N>1 path's host-side logic: LPT sharding of a
batch by the planner's per-subdomain costs (bench.setup_problem, the default multi-GPU mode), and the
additive all-reduce of per-rank partial dual vectors q = sum_i scatter(F_i gather(lambda)) through
the product's SCPlan.apply_global.  Without a GPU the per-rank partial of
sc_apply is supplied by the oracle; the GPU partial itself is checked against the same oracle sum in
tests/test_gpu_parity.py::test_apply_matches_oracle_sum."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_21037_b200 import SCPlan
from paper_2509_21037_b200.shard import imbalance, lpt_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from synth import config_problem
    P = config_problem("cfg1")
    costs = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1).subdomain_costs()
    parts = lpt_partition(costs, world)
    mine = parts[rank]
    rng = np.random.default_rng(42)
    lam = rng.standard_normal(P.n_lambda)
    q = np.zeros(P.n_lambda)
    for i in mine:
        sd = P.subdomains[i]
        q[sd.lambda_map] += oracle.subdomain_F(sd) @ lam[sd.lambda_map]
    qt = torch.from_numpy(q)
    dist.all_reduce(qt, op=dist.ReduceOp.SUM)
    # every rank agrees on the partition
    sizes = torch.tensor([len(mine)], dtype=torch.int64)
    allsz = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allsz, sizes)
    if rank == 0:
        out.put((qt.numpy().copy(), [int(s.item()) for s in allsz], parts, list(costs)))
    dist.barrier()
    dist.destroy_process_group()


def test_lpt_partition_properties():
    rng = np.random.default_rng(0)
    costs = rng.uniform(1, 3, 512)
    for k in (1, 2, 4, 8):
        parts = lpt_partition(costs, k)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(512))
        assert imbalance(costs, parts) < 1.01
    assert lpt_partition([5.0, 1.0, 1.0, 1.0, 1.0, 1.0], 2) == [[0], [1, 2, 3, 4, 5]]


def test_two_rank_sharded_apply_allreduce_equals_global():
    import oracle
    from synth import config_problem
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    q, sizes, parts, costs = out.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    P = config_problem("cfg1")
    assert sum(sizes) == len(P.subdomains)
    assert sorted(i for p in parts for i in p) == list(range(len(P.subdomains)))
    assert imbalance(costs, parts) < 1.15
    lam = np.random.default_rng(42).standard_normal(P.n_lambda)
    q_ref = np.zeros(P.n_lambda)
    for sd in P.subdomains:
        q_ref[sd.lambda_map] += oracle.subdomain_F(sd) @ lam[sd.lambda_map]
    assert np.linalg.norm(q - q_ref) <= 1e-12 * np.linalg.norm(q_ref)


def _worker_apply_global(rank, world, port, out):
    """Each rank: its LPT shard of cfg1 (bench.setup_problem), a host-only plan of the shard, the
    rank's partial q from the oracle in place of sc_apply, then SCPlan.apply_global (the product's
    collective path: all-reduce SUM of the partials)."""
    import argparse
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import bench
    P, info = bench.setup_problem(argparse.Namespace(weak=False, perturbed=False), "cfg1", world, rank)
    plan = SCPlan(P.subdomains, n_lambda=P.n_lambda, device=-1)
    lam = np.random.default_rng(9).standard_normal(P.n_lambda)

    def partial(lam_t, q_t, stream=None):
        qq = np.zeros(P.n_lambda)
        for sd in P.subdomains:
            qq[sd.lambda_map] += oracle.subdomain_F(sd) @ lam_t.numpy()[sd.lambda_map]
        q_t.copy_(torch.from_numpy(qq))

    plan.apply = partial
    q = torch.zeros(P.n_lambda, dtype=torch.float64)
    plan.apply_global(torch.from_numpy(lam), q)
    ids = torch.tensor([sd.id for sd in P.subdomains] + [-1] * (16 - len(P.subdomains)), dtype=torch.int64)
    allids = [torch.zeros(16, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allids, ids)
    if rank == 0:
        out.put((q.numpy().copy(), [a.tolist() for a in allids], info))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_apply_global_product_path():
    import oracle
    from synth import config_problem
    world = 2
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_apply_global, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    q, ids, info = out.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    P = config_problem("cfg1")
    got = sorted(i for r in ids for i in r if i >= 0)
    assert got == list(range(len(P.subdomains)))  # every subdomain on exactly one rank
    assert info["nsub_total"] == len(P.subdomains) and sum(info["nsub_per_rank"]) == len(P.subdomains)
    lam = np.random.default_rng(9).standard_normal(P.n_lambda)
    q_ref = np.zeros(P.n_lambda)
    for sd in P.subdomains:
        q_ref[sd.lambda_map] += oracle.subdomain_F(sd) @ lam[sd.lambda_map]
    assert np.linalg.norm(q - q_ref) <= 1e-12 * np.linalg.norm(q_ref)
