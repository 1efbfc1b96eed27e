"""Subdomain -> GPU assignment: subdomains are independent units,
so a batch is partitioned over ranks by longest-processing-time-first on the planner's per-subdomain
cost (executed FP64 flops), with no collective on the assembly path."""
from __future__ import annotations

import heapq
from typing import List, Sequence


def lpt_partition(costs: Sequence[float], nparts: int) -> List[List[int]]:
    """Greedy LPT: largest cost first onto the currently lightest part.  Deterministic (ties by
    index); each part's indices are returned ascending."""
    if nparts < 1:
        raise ValueError("nparts must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    heap = [(0.0, p) for p in range(nparts)]
    parts: List[List[int]] = [[] for _ in range(nparts)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(i)
        heapq.heappush(heap, (load + float(costs[i]), p))
    return [sorted(p) for p in parts]


def imbalance(costs: Sequence[float], parts: List[List[int]]) -> float:
    """max part load / mean part load (1.0 = perfect)."""
    loads = [sum(float(costs[i]) for i in p) for p in parts]
    mean = sum(loads) / max(len(loads), 1)
    return max(loads) / mean if mean > 0 else 1.0
