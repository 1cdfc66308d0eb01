"""The N > 1 path on CPU: two gloo ranks shard the sample indices of a level,
evaluate their shard (here with the C oracle standing in for the device
evaluator) and combine the per-level sums with one allreduce; the result must
equal the single-process fold and the reference's moments."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2106_11117_b200 import shard

N = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import oracle_py
    from paper_2106_11117_b200 import configs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard.shard_range(N, rank, world)
    orc = oracle_py.COracle()
    d = configs.config0()
    mesh = oracle_py.MeshArrays(*configs.build_mesh(d).arrays())
    rc, dq, q, _, _ = orc.eval_pairs(mesh, oracle_py.problem(d.dt, d.substeps), None, None, 0, 0, first, count)
    assert rc == 0
    local = {"n_samples": count, "sum_dq": float(np.sum(dq)), "sum_dq2": float(np.sum(dq * dq)),
             "sum_q": float(np.sum(q)), "sum_q2": float(np.sum(q * q))}
    res = shard.allreduce_level_sums([local])
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, count, q.tolist()))
    if rank == 0:
        out.put((res, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_every_index_once():
    for n in (1, 7, 256, 65536):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b
            assert spans[-1][0] + spans[-1][1] == n
    with pytest.raises(ValueError):
        shard.shard_range(4, 2, 2)
    # whole 64-sample granules: config-1 level 4 (256 samples) at 8 ranks
    spans = [shard.shard_range(256, r, 8) for r in range(8)]
    assert all(c in (0, 64) for _, c in spans) and sum(c for _, c in spans) == 256


def test_shard_levels_balance_whole_granules():
    from paper_2106_11117_b200 import configs
    counts = configs.CONFIG1_COUNTS
    costs = [1.0, 2.0, 2.5, 5.0, 12.0]  # pair costs grow with the level
    for world in (1, 2, 4, 8):
        plan = shard.shard_levels(counts, costs, world)
        for lvl, n in enumerate(counts):
            spans = [plan[r][lvl] for r in range(world)]
            assert spans[0][0] == 0 and sum(c for _, c in spans) == n
            for (a, c), (b, _) in zip(spans, spans[1:]):
                assert a + c == b
            assert all(c % 64 == 0 or a + c == n for a, c in spans)
        work = [sum(plan[r][l][1] * costs[l] for l in range(len(counts))) for r in range(world)]
        assert max(work) / (sum(work) / world) < 1.1


def test_two_gloo_ranks_match_single_process(golden):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res, gathered = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    lv = res[0]
    assert lv["n_samples"] == N
    # per-sample values are independent of the sharding (index-keyed streams)
    q = np.concatenate([np.array(g[2]) for g in sorted(gathered)])
    ref = golden("config0_samples.json")["lts"]["q"][:N]
    assert np.max(np.abs(q - ref) / np.abs(ref)) < 1e-12
    # the reduced sums equal the one-process fold of the same values
    assert lv["sum_q"] == pytest.approx(float(np.sum(ref)), rel=1e-12)
    assert lv["sum_q2"] == pytest.approx(float(np.sum(np.square(ref))), rel=1e-12)
    single = shard.estimators({"n_samples": N, "sum_dq": float(np.sum(ref)), "sum_dq2": float(np.sum(np.square(ref))),
                               "sum_q": float(np.sum(ref)), "sum_q2": float(np.sum(np.square(ref)))})
    assert lv["variance"] == pytest.approx(single["variance"], rel=1e-9)
