"""BASELINE configs at their stated sizes against the unmodified reference
(golden fixtures from oracle/_ref via oracle/make_golden.py --only-round2 /
--only-config1-full), through the C ABI on the device:

* config 0 at its BASELINE 1024 samples: per-sample Q and the level moments;
* config 1 per-level sums, means and variances at the BASELINE N_l
  (65536 / 16384 / 4096 / 1024 / 256 coupled pairs);
* config 1's global leap-frog comparison arm (dt = 0.2 h_min on every level,
  reference leapfrog_step, src/integrators.cpp:89-115);
* config 3's mesh (h = 1/1024, square at h/8, p = 8, |R| = 1.06 M) with the
  horizon cut to 16 / 40 global steps (reference lts_step,
  src/integrators.cpp:117-157), on the BASELINE QoI and on a QoI over the
  refined square (the BASELINE box is outside the square's domain of
  dependence for such short horizons);
* the device-resident leg: the device moment fold against the host fold, and
  instability reporting through wmc_synchronize.

Tolerances (BASELINE north_star): per-sample QoI 1e-10 relative, per-level
means and variances 1e-9 relative."""
import os

import numpy as np
import pytest

from paper_2106_11117_b200 import configs, wavemc
from paper_2106_11117_b200._native import WMC_LEAPFROG

pytestmark = pytest.mark.gpu

QOI_RTOL = 1e-10
MOMENT_RTOL = 1e-9
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def per_sample_rel(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


def test_config0_baseline_1024_samples_and_moments(golden):
    g = golden("config0_moments_1024.json")["levels"][0]
    assert g["N"] == configs.CONFIG0_COUNT
    lv = configs.build_level(configs.config0())
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, g["N"])
    assert per_sample_rel(qf, g["q"]) < QOI_RTOL
    st = wavemc.run_mlmc_fixed([lv], [g["N"]], seed=0)[0]
    assert st["n_samples"] == g["N"]
    for k in ("sum_dq", "sum_q", "sum_dq2", "sum_q2", "mean_dq", "variance", "mc_variance"):
        assert st[k] == pytest.approx(g[k], rel=MOMENT_RTOL), k


def test_config1_global_leapfrog_pairs_match_reference(golden):
    g = golden("config1_lf_pairs.json")
    defs = configs.config1("lf")
    assert defs[0].dt == pytest.approx(g["dt"], rel=1e-15)
    levels = [configs.build_level(d) for d in defs]
    for lv in g["levels"]:
        l, n = lv["level"], lv["N"]
        assert levels[l].info["n_steps"] == lv["n_steps"]
        dq, qf, cost = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l
        # LF: n_steps full products per solve (StepCounters, integrators.cpp:94)
        assert cost["matvec_full"] == n * lv["n_steps"] * (2 if l else 1)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "config1_full_moments.json")),
                    reason="config1_full_moments.json not generated")
def test_config1_moments_at_baseline_counts_match_reference(golden):
    g = golden("config1_full_moments.json")
    counts = [lv["N"] for lv in g["levels"]]
    assert counts == configs.CONFIG1_COUNTS
    levels = [configs.build_level(d) for d in configs.config1()]
    stats = wavemc.run_mlmc_fixed(levels, counts, seed=0)
    for st, want in zip(stats, g["levels"]):
        assert st["n_samples"] == want["N"]
        for k in ("mean_dq", "variance", "mc_variance", "sum_dq", "sum_q", "sum_dq2", "sum_q2"):
            assert st[k] == pytest.approx(want[k], rel=MOMENT_RTOL), (want["level"], k)


@pytest.fixture(scope="module")
def config3_mesh():
    return configs.build_mesh(configs.config3())


@pytest.mark.parametrize("case", ["baseline_box", "square_box", "square_box_long"])
def test_config3_samples_match_reference(golden, config3_mesh, case):
    g = golden("config3_samples.json")
    d = configs.config3()
    if case == "baseline_box":
        T, box, idx, want = g["T"], (0.7, 0.9, 0.4, 0.6), g["index"], g["q"]
        hdr = g["header"]
    else:
        c = g[case]
        T, box, want, hdr = c["T"], tuple(c["box"]), c["q"], c["header"]
        idx = list(range(c["first"], c["first"] + len(want)))
    spec = wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, final_time=T, qoi_box=box, batch=64)
    lv = wavemc.Level(config3_mesh, spec)
    assert lv.info["n"] == int(hdr["n"]) and lv.info["n_r"] == int(hdr["n_r"])
    assert lv.info["n_steps"] == int(hdr["n_steps"])
    assert lv.info["substep_path"] == 5  # the temporally blocked tiled step
    got = []
    for i in idx:  # contiguous runs
        _, q, _ = wavemc.eval_pairs(lv, None, 0, 0, i, 1)
        got.append(q[0])
    assert per_sample_rel(got, want) < QOI_RTOL, (case, lv.info.get("substep_path"))


def test_moments_device_matches_host_fold():
    import torch
    levels = [configs.build_level(d, batch=512) for d in configs.config1()[:3]]
    n = 700
    for l, lv in enumerate(levels):
        coarse = levels[l - 1] if l else None
        dq, qf, _ = wavemc.eval_pairs(lv, coarse, 0, l, 11, n)
        d_dq = torch.tensor(dq, dtype=torch.float64, device="cuda")
        d_q = torch.tensor(qf, dtype=torch.float64, device="cuda")
        out = torch.zeros(4, dtype=torch.float64, device="cuda")
        wavemc.moments_device(lv, d_dq.data_ptr(), d_q.data_ptr(), n, out.data_ptr())
        wavemc.synchronize(lv)
        got = out.cpu().numpy()
        host = wavemc.run_mlmc_fixed(levels[:l + 1], [0] * l + [n], seed=0, first=[0] * l + [11])[l]
        for k, key in enumerate(("sum_dq", "sum_dq2", "sum_q", "sum_q2")):
            assert got[k] == pytest.approx(host[key], rel=1e-12, abs=1e-300), (l, key)


def test_moments_device_refuses_qoi_vectors(mesh1d):
    import torch
    lv = wavemc.Level.experiment("smooth1d", 0, mesh1d("smooth1d")[0])
    assert lv.info["nq"] > 1
    buf = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(wavemc.ConfigError):
        wavemc.moments_device(lv, buf.data_ptr(), buf.data_ptr(), 2, buf.data_ptr())


def test_device_resident_path_reports_instability():
    """wmc_eval_pairs_device + wmc_synchronize report the first failing
    sample and its step exactly like the host path (finish_pairs)."""
    import torch
    lv = wavemc.Level(configs.build_mesh(configs.config0()),
                      wavemc.LevelSpec(dt=0.2, final_time=20.0, integrator=WMC_LEAPFROG))
    with pytest.raises(wavemc.NumericalError) as host:
        wavemc.eval_pairs(lv, None, 0, 0, 5, 3)
    d_dq = torch.empty(3, dtype=torch.float64, device="cuda")
    d_q = torch.empty(3, dtype=torch.float64, device="cuda")
    wavemc.eval_pairs_device(lv, None, 0, 0, 5, 3, d_dq.data_ptr(), d_q.data_ptr())
    with pytest.raises(wavemc.NumericalError) as dev:
        wavemc.synchronize(lv)
    assert (dev.value.sample, dev.value.step) == (host.value.sample, host.value.step) == (5, host.value.step)
    wavemc.synchronize(lv)  # the record was cleared
    # a stable level leaves it clean
    ok = configs.build_level(configs.config0())
    d_dq = torch.empty(64, dtype=torch.float64, device="cuda")
    d_q = torch.empty(64, dtype=torch.float64, device="cuda")
    wavemc.eval_pairs_device(ok, None, 0, 0, 0, 64, d_dq.data_ptr(), d_q.data_ptr())
    wavemc.synchronize(ok)


def test_config3_tiled_step_matches_hbm_resident_substeps(config3_mesh, monkeypatch):
    """The tiled step (R in spatial tiles, substeps on chip) against the
    HBM-resident substep kernels on the config-3 mesh, a batch of 64 samples
    at 12 global steps (every tile, both region shapes, every sample)."""
    d = configs.config3()
    spec = wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, final_time=12 * d.dt,
                            qoi_box=(0.4375, 0.5625, 0.4375, 0.5625), batch=64)
    tiled = wavemc.Level(config3_mesh, spec)
    monkeypatch.setenv("WMC_TILED", "0")
    glob = wavemc.Level(config3_mesh, spec)
    monkeypatch.delenv("WMC_TILED")
    assert tiled.info["substep_path"] == 5 and glob.info["substep_path"] == 3
    _, a, _ = wavemc.eval_pairs(tiled, None, 0, 0, 100, 64)
    _, b, _ = wavemc.eval_pairs(glob, None, 0, 0, 100, 64)
    assert per_sample_rel(a, b) < QOI_RTOL


@pytest.mark.parametrize("lvl", [3, 4])
def test_tiled_step_on_config1_levels(lvl, monkeypatch):
    """Config-1 levels 3 (p = 4) and 4 (p = 2): the tiled step against the
    lattice / HBM-resident paths and, for pairs, the reference goldens."""
    d = configs.config1()[lvl]
    monkeypatch.setenv("WMC_SUBSTEP_PATH", "tiled")
    tiled = configs.build_level(d)
    monkeypatch.setenv("WMC_SUBSTEP_PATH", "global")
    monkeypatch.setenv("WMC_TILED", "0")
    other = configs.build_level(d)
    monkeypatch.delenv("WMC_SUBSTEP_PATH")
    monkeypatch.delenv("WMC_TILED")
    assert tiled.info["substep_path"] == 5 and other.info["substep_path"] == 3
    assert configs.build_level(d).info["substep_path"] != 5  # small boxes keep the halo-free paths
    _, a, _ = wavemc.eval_pairs(tiled, None, 0, lvl, 0, 96)
    _, b, _ = wavemc.eval_pairs(other, None, 0, lvl, 0, 96)
    assert per_sample_rel(a, b) < QOI_RTOL


@pytest.mark.parametrize("n_coarse", [128, 256])
def test_tiled_step_with_streamed_slabs_on_mid_size_boxes(n_coarse, monkeypatch):
    """Refined boxes of 129^2 / 257^2 nodes at p = 8: thin side bands, square
    corner tiles and one streamed slab (128- and 256-thread CTAs) against the
    HBM-resident substeps, with the QoI over the refined square."""
    d = configs.LevelDef(n_coarse, 8, 0.2 / n_coarse, 8, configs.config1()[0].integrator)
    mesh = configs.build_mesh(d)
    spec = wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, final_time=20 * d.dt,
                            qoi_box=(0.4375, 0.5625, 0.4375, 0.5625), batch=64)
    plan = wavemc.tile_plan(mesh, spec)
    assert plan["ok"] and plan["layout"].endswith("+thin+stream") and plan["n_slabs"] >= 1
    monkeypatch.setenv("WMC_SUBSTEP_PATH", "tiled")
    tiled = wavemc.Level(mesh, spec)
    monkeypatch.setenv("WMC_SUBSTEP_PATH", "global")
    monkeypatch.setenv("WMC_TILED", "0")
    other = wavemc.Level(mesh, spec)
    monkeypatch.delenv("WMC_SUBSTEP_PATH")
    monkeypatch.delenv("WMC_TILED")
    assert tiled.info["substep_path"] == 5 and other.info["substep_path"] == 3
    _, a, _ = wavemc.eval_pairs(tiled, None, 0, 0, 7, 70)
    _, b, _ = wavemc.eval_pairs(other, None, 0, 0, 7, 70)
    assert per_sample_rel(a, b) < QOI_RTOL
