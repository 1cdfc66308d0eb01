"""The reference's own 1D sampling experiments on the device (SURVEY.md
section 8(f) row 2): smooth1d (KL field) and jump1d (jump field), LF-LTS and
LF, per-sample CFL step, Neumann, 512-point QoI vectors -- against the
unmodified reference through its make_problem (tests/golden/experiments.json):
per-sample QoI vectors within 1e-10 (relative to the vector's size) and the
adaptive run_mlmc with the same N_l and estimate."""
import numpy as np
import pytest

from paper_2106_11117_b200 import wavemc
from paper_2106_11117_b200._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING

pytestmark = pytest.mark.gpu

CASES = ["smooth1d_lts", "smooth1d_lf", "jump1d_lts", "jump1d_lf"]


def _levels(case, mesh1d, n=5):
    name, kind = case.split("_")
    integ = WMC_LOCAL_TIME_STEPPING if kind == "lts" else WMC_LEAPFROG
    meshes = mesh1d(name)
    return [wavemc.Level.experiment(name, l, meshes[l], integ) for l in range(n)], integ


def _weights(nq):
    w = np.full(nq, 6.0 / (nq - 1))
    w[0] = w[-1] = 0.5 * 6.0 / (nq - 1)
    return w


@pytest.mark.parametrize("case", CASES)
def test_experiment_pairs_match_reference(golden, case, mesh1d):
    g = golden("experiments.json")[case]
    levels, _ = _levels(case, mesh1d, 3)
    w = _weights(512)
    for lv in g["levels"]:
        l, first, ref = lv["level"], lv["first"], lv["samples"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, first, len(ref))
        assert dq.shape == (len(ref), 512)
        for i, r in enumerate(ref):
            scale = max(np.max(np.abs(r["q_every4"])), 1e-300)
            assert np.max(np.abs(qf[i, ::4] - r["q_every4"])) < 1e-10 * scale, (l, i)
            assert np.max(np.abs(dq[i, ::4] - r["dq_every4"])) < 2e-10 * scale, (l, i)
            assert np.sqrt(np.sum(w * qf[i] ** 2)) == pytest.approx(r["q_norm"], rel=1e-10)
            assert np.sqrt(np.sum(w * dq[i] ** 2)) == pytest.approx(r["dq_norm"], rel=1e-9, abs=1e-12 * r["q_norm"])


@pytest.mark.parametrize("case", CASES)
def test_experiment_adaptive_mlmc_matches_reference(golden, case, mesh1d):
    g = golden("experiments.json")[case]
    levels, integ = _levels(case, mesh1d)
    name = case.split("_")[0]
    cost = wavemc.experiment_model_cost(name, integ)
    a = g["adaptive"]
    res = wavemc.run_mlmc(levels, cost, wavemc.MlmcConfig(eps=a["eps"], max_level=4))
    assert res.converged == a["converged"]
    assert [s["n_samples"] for s in res.levels] == [lv["N"] for lv in a["levels"]]
    assert res.estimate == pytest.approx(a["estimate_norm"], rel=1e-9)
    assert np.max(np.abs(res.estimate_vector[::4] - a["estimate_every4"])) < 1e-9 * a["estimate_norm"]
    for s, lv in zip(res.levels, a["levels"]):
        assert s["variance"] == pytest.approx(lv["variance"], rel=1e-9)
        assert s["mean_dq"] == pytest.approx(lv["mean_dq_norm"], rel=1e-9)


@pytest.mark.parametrize("case", ["smooth1d_lts", "jump1d_lf"])
def test_fused_small_solve_is_bitwise_the_batched_path(case, mesh1d):
    """Small batches take the fused one-CTA-per-sample solve; it repeats the
    batched kernels' arithmetic exactly (same bits either way)."""
    levels, _ = _levels(case, mesh1d, 2)
    fused = wavemc.eval_pairs(levels[1], levels[0], 3, 1, 10, 40)  # 40 <= 2 x SMs: fused solve
    big = wavemc.eval_pairs(levels[1], levels[0], 3, 1, 0, 600)  # one batch of 600: batched kernels
    assert np.array_equal(fused[0], big[0][10:50]) and np.array_equal(fused[1], big[1][10:50])
