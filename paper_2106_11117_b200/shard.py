"""Sample sharding across GPUs and the one exchange step.

Rank r of G evaluates indices [r N / G, (r+1) N / G) of every level; the
streams are keyed by the global index (RngStream(seed, level, index),
reference src/rng.cpp:14-32), so every per-sample result is independent of G.
The only collective is the allreduce of the per-level LevelAccumulator sums
(reference include/wavemc/mlmc.hpp:53-66); the estimators are then formed
exactly as estimate_variance / estimate_mc_variance (src/mlmc.cpp:61-73).
"""
from __future__ import annotations

import math

SUM_KEYS = ("n_samples", "sum_dq", "sum_dq2", "sum_q", "sum_q2")


GRANULE = 64  # samples per batch lane group of the device kernels


def shard_range(n: int, rank: int, world: int, granule: int = GRANULE) -> tuple[int, int]:
    """(first, count) of rank's contiguous share of n indices, in whole
    granules of `granule` samples (the device batch granule: no rank pads a
    partial batch except the one holding the level's tail)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    g = (n + granule - 1) // granule
    g0, g1 = rank * g // world, (rank + 1) * g // world
    a, b = min(n, granule * g0), min(n, granule * g1)
    return a, b - a


def shard_levels(counts: list[int], pair_costs: list[float], world: int,
                 granule: int = GRANULE) -> list[list[tuple[int, int]]]:
    """Per rank, per level: (first, count) in whole granules, balanced over
    all levels: each level's granules split evenly and its remainder granules
    go to the ranks with the least work so far (cost = pair cost x samples);
    every rank's indices of a level stay contiguous, ranks in order."""
    load = [0.0] * world
    out = [[(0, 0)] * len(counts) for _ in range(world)]
    for lvl in sorted(range(len(counts)), key=lambda q: -pair_costs[q] * counts[q]):
        n = counts[lvl]
        g = (n + granule - 1) // granule
        per = [g // world] * world
        for r in sorted(range(world), key=lambda q: (load[q], q))[: g % world]:
            per[r] += 1
        first = 0
        for r in range(world):
            a, b = min(n, granule * first), min(n, granule * (first + per[r]))
            out[r][lvl] = (a, b - a)
            load[r] += (b - a) * pair_costs[lvl]
            first += per[r]
    return out


def estimators(sums: dict) -> dict:
    """Reference estimate_variance / estimate_mc_variance on folded sums."""
    n = sums["n_samples"]
    out = dict(sums)
    if n >= 2:
        sn = math.sqrt(sums["sum_dq"] ** 2)
        qn = math.sqrt(sums["sum_q"] ** 2)
        out["variance"] = max(0.0, (sums["sum_dq2"] - sn * sn / n) / (n - 1.0))
        out["mc_variance"] = max(0.0, (sums["sum_q2"] - qn * qn / n) / n)
    else:
        out["variance"] = out["mc_variance"] = 0.0
    out["mean_dq"] = sums["sum_dq"] * (1.0 / n) if n else 0.0
    return out


def allreduce_level_sums(per_level: list[dict], device=None) -> list[dict]:
    """Sum the per-level accumulators over all ranks (one allreduce of
    5 doubles per level) and recompute the estimators."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([[float(s[k]) for k in SUM_KEYS] for s in per_level], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
    rows = t.cpu().tolist()
    out = []
    for lvl, row in enumerate(rows):
        sums = dict(zip(SUM_KEYS, row))
        sums["n_samples"] = int(round(sums["n_samples"]))
        sums["level"] = lvl
        out.append(estimators(sums))
    return out
