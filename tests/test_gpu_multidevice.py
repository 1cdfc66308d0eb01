"""The multi-GPU paths on the one device of this box:

* the C-ABI multi-device drivers (wmc_run_mlmc_fixed_multi /
  wmc_run_mlmc_multi) with two device groups -- two level sets, both on
  device 0, each on its own host thread -- must give the one-device results
  bitwise (64-sample granules per group, host fold in index order);
* the sharded rank path of bench.py: two processes (gloo ranks, both on
  device 0: independent kernels, nothing waits on another rank's kernel)
  evaluate their whole-granule shards of every level and combine the
  per-level sums with one allreduce; per-sample results bitwise equal to one
  process, moments within 1e-12."""
import os
import socket

import numpy as np
import pytest

from paper_2106_11117_b200 import configs, shard, wavemc

pytestmark = pytest.mark.gpu

COUNTS = [700, 300, 130]


def _levels():
    return [configs.build_level(d, batch=256) for d in configs.config1()[:3]]


def test_multi_device_fixed_driver_is_bitwise_the_single_device_one():
    one = _levels()
    two = [_levels(), _levels()]
    a = wavemc.run_mlmc_fixed(one, COUNTS, seed=0)
    b = wavemc.run_mlmc_fixed_multi(two, COUNTS, seed=0)
    for x, y in zip(a, b):
        for k in ("n_samples", "sum_dq", "sum_dq2", "sum_q", "sum_q2", "variance", "mc_variance", "mean_dq"):
            assert x[k] == y[k], k
        assert x["cost"] == y["cost"]


def test_multi_device_adaptive_driver_matches_run_mlmc(golden):
    g = golden("config1_adaptive.json")
    one = [configs.build_level(d) for d in configs.config1()]
    two = [[configs.build_level(d) for d in configs.config1()] for _ in range(2)]
    cfg = wavemc.MlmcConfig(eps=g["eps"])
    r1 = wavemc.run_mlmc(one, g["model_cost"], cfg)
    r2 = wavemc.run_mlmc_multi(two, g["model_cost"], cfg)
    assert [s["n_samples"] for s in r1.levels] == [s["n_samples"] for s in r2.levels] == [lv["N"] for lv in g["levels"]]
    assert r1.estimate == r2.estimate and r1.total_variance == r2.total_variance and r1.bias == r2.bias


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2106_11117_b200 import configs, shard, wavemc
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    levels = [configs.build_level(d, batch=256) for d in configs.config1()[:3]]
    costs = [lv.info["dof_updates_per_solve"] for lv in levels]
    pair = [costs[l] + (costs[l - 1] if l else 0.0) for l in range(3)]
    plan = shard.shard_levels(COUNTS, pair, world)[rank]
    stats = wavemc.run_mlmc_fixed(levels, [c for _, c in plan], 0, [f for f, _ in plan])
    summed = shard.allreduce_level_sums(stats)
    per_sample = []
    for l, (f, c) in enumerate(plan):
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, f, c) if c else ([], [], None)
        per_sample.append((f, list(map(float, dq)), list(map(float, qf))))
    gathered = [None] * world
    dist.all_gather_object(gathered, per_sample)
    if rank == 0:
        out.put((summed, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gloo_ranks_match_one_process():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    summed, gathered = out.get(timeout=900)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    levels = _levels()
    ref = wavemc.run_mlmc_fixed(levels, COUNTS, seed=0)
    for l in range(3):
        dq_ref, qf_ref, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, COUNTS[l])
        parts = sorted((g[l] for g in gathered), key=lambda t: t[0])
        dq = np.concatenate([np.array(p[1]) for p in parts])
        qf = np.concatenate([np.array(p[2]) for p in parts])
        assert np.array_equal(dq, dq_ref) and np.array_equal(qf, qf_ref), l  # index-keyed streams
        assert summed[l]["n_samples"] == COUNTS[l]
        for k in ("sum_dq", "sum_dq2", "sum_q", "sum_q2", "variance", "mean_dq"):
            assert summed[l][k] == pytest.approx(ref[l][k], rel=1e-12, abs=1e-300), (l, k)
