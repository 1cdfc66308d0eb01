"""The reference's narrow-channel experiment on the device (SURVEY.md section
8(f) row 2, make_problem Channel2d, src/experiments.cpp:108-172): per-sample
geometry (channel width b ~ U[0.001, 0.007] moving the mesh), Neumann,
per-sample CFL step with warm starts, bump u0, QoI u(T) on the line
x = -0.4 -- against the unmodified reference on a small hierarchy
(tests/golden/channel: the reference meshes of levels 0..2 and its
per-sample QoI vectors, cost records and run_mlmc, oracle/make_golden.py
--only-channel): per-sample QoI vectors within 1e-10 relative to the
vector's size, identical cost records, the adaptive run with the same N_l."""
import os

import numpy as np
import pytest

from paper_2106_11117_b200 import wavemc
from paper_2106_11117_b200._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "channel")


@pytest.fixture(scope="module")
def channel_golden():
    import json
    with open(os.path.join(GOLDEN, "channel.json")) as f:
        return json.load(f)


def _levels(g, kind):
    c = g["config"]
    integ = WMC_LOCAL_TIME_STEPPING if kind == "lts" else WMC_LEAPFROG
    meshes = [wavemc.Mesh.load(os.path.join(GOLDEN, f"mesh_l{l}.txt.gz")) for l in range(c["max_level"] + 1)]
    ov = dict(h0=c["h0"], fine_h=c["fine_h"], max_level=c["max_level"], grid_n=c["grid_n"])
    return [wavemc.Level.channel(m, l, integ, **ov) for l, m in enumerate(meshes)], integ, ov


@pytest.mark.parametrize("kind", ["lts", "lf"])
def test_channel_pairs_match_reference(channel_golden, kind):
    g = channel_golden
    levels, integ, ov = _levels(g, kind)
    assert wavemc.experiment_model_cost("channel2d", integ, **ov) == pytest.approx(g[kind]["model_cost"], rel=1e-15)
    nq = g["config"]["grid_n"]
    for lv in g[kind]["levels"]:
        l, first, ref = lv["level"], lv["first"], lv["samples"]
        dq, qf, cost = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, first, len(ref))
        assert dq.shape == (len(ref), nq)
        for i, r in enumerate(ref):
            q_ref, dq_ref = np.array(r["q"]), np.array(r["dq"])
            scale = np.max(np.abs(q_ref))
            assert np.max(np.abs(qf[i] - q_ref)) < 1e-10 * scale, (l, i, np.max(np.abs(qf[i] - q_ref)) / scale)
            assert np.max(np.abs(dq[i] - dq_ref)) < 2e-10 * scale, (l, i)
        want = np.sum([r["cost"] for r in ref], axis=0)
        got = [cost["matvec_full"], cost["matvec_fine"], cost["matvec_coarse"], cost["weighted_work"]]
        assert got == want.tolist(), (l, got, want)


@pytest.mark.parametrize("kind", ["lts", "lf"])
def test_channel_adaptive_mlmc_matches_reference(channel_golden, kind):
    g = channel_golden
    levels, integ, ov = _levels(g, kind)
    a = g[kind]["adaptive"]
    cost = wavemc.experiment_model_cost("channel2d", integ, **ov)
    res = wavemc.run_mlmc(levels, cost, wavemc.MlmcConfig(eps=a["eps"], max_level=g["config"]["max_level"]))
    assert res.converged == a["converged"]
    assert [s["n_samples"] for s in res.levels] == [lv["N"] for lv in a["levels"]]
    assert res.estimate == pytest.approx(a["estimate_norm"], rel=1e-9)
    assert np.max(np.abs(res.estimate_vector - a["estimate"])) < 1e-9 * a["estimate_norm"]
    for s, lv in zip(res.levels, a["levels"]):
        assert s["variance"] == pytest.approx(lv["variance"], rel=1e-9)
        assert s["mean_dq"] == pytest.approx(lv["mean_dq_norm"], rel=1e-9)


def test_channel_batches_are_bitwise_invariant(channel_golden):
    levels, _, _ = _levels(channel_golden, "lts")
    a = wavemc.eval_pairs(levels[1], levels[0], 5, 1, 0, 130)
    b = wavemc.eval_pairs(levels[1], levels[0], 5, 1, 40, 30)
    assert np.array_equal(a[1][40:70], b[1]) and np.array_equal(a[0][40:70], b[0])
