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


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous share of n indices."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    a, b = rank * n // world, (rank + 1) * n // world
    return a, b - a


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
