"""Per-sample CFL step on the device: the
batched power iteration and per-sample dt / step count against the unmodified
reference's stable_dt recipe (src/experiments.cpp:30-43 over max_eigenvalue /
coarse_max_eigenvalue, src/fem.cpp:132-189; golden vectors from
oracle/make_golden.py --only-cfl) and the C restatement.  Samples of one batch
run different step counts; each keeps its own horizon."""
import numpy as np
import pytest

from oracle_py import MeshArrays, problem
from paper_2106_11117_b200 import configs, wavemc

pytestmark = pytest.mark.gpu

QOI_RTOL = 1e-10


def per_sample_rel(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


def _level(d, safety, **kw):
    spec = configs.level_spec(d)
    spec.cfl_safety = safety
    for k, v in kw.items():
        setattr(spec, k, v)
    return wavemc.Level(configs.build_mesh(d), spec)


def test_config0_cfl_matches_reference(golden):
    g = golden("cfl_samples.json")
    d = configs.config0()
    lv = _level(d, g["safety"])
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, len(g["config0_lts"]["q"]))
    assert per_sample_rel(qf, g["config0_lts"]["q"]) < QOI_RTOL
    lf = _level(configs.config0_leapfrog(), g["safety"])
    _, qf, _ = wavemc.eval_pairs(lf, None, 0, 0, 0, len(g["config0_lf"]["q"]))
    assert per_sample_rel(qf, g["config0_lf"]["q"]) < QOI_RTOL


def test_config1_cfl_pairs_match_reference(golden):
    g = golden("cfl_samples.json")
    defs = configs.config1()[:3]
    levels = [_level(d, g["safety"]) for d in defs]
    for lv in g["config1_pairs"]["levels"]:
        l, n = lv["level"], lv["N"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l


@pytest.mark.parametrize("path", ["global", "onchip"])
def test_cfl_substep_paths_agree(golden, path, monkeypatch):
    g = golden("cfl_samples.json")
    monkeypatch.setenv("WMC_SUBSTEP_PATH", path)
    lv = _level(configs.config0(), g["safety"])
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, len(g["config0_lts"]["q"]))
    assert per_sample_rel(qf, g["config0_lts"]["q"]) < QOI_RTOL


def test_cfl_batches_are_bitwise_invariant():
    d = configs.config0()
    a = _level(d, 0.9, batch=64)
    b = _level(d, 0.9)
    _, qa, _ = wavemc.eval_pairs(a, None, 0, 0, 0, 150)
    _, qb, _ = wavemc.eval_pairs(b, None, 0, 0, 0, 150)
    _, qc, _ = wavemc.eval_pairs(b, None, 0, 0, 50, 60)
    assert np.array_equal(qa, qb) and np.array_equal(qa[50:110], qc)


def test_cfl_many_samples_match_c_oracle(coracle):
    """A full batch (step counts differ across its samples) spot-checked."""
    d = configs.config1()[0]
    lv = _level(d, 0.9)
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, 512)
    ma = MeshArrays(*configs.build_mesh(d).arrays())
    pb = problem(d.dt, d.substeps, 1, cfl_safety=0.9)
    steps = set()
    for i in (0, 1, 63, 200, 511):
        cells = coracle.draw_cells(0, 0, i)
        rc, q, _, _ = coracle.solve(ma, pb, cells)
        assert rc == 0 and abs(qf[i] - q) < QOI_RTOL * abs(q), i
        rc, dt, _ = coracle.stable_dt(ma, pb, cells)
        steps.add(int(np.ceil(1.0 / dt - 1e-12)))
    assert len(steps) > 1  # the batch really mixes horizons


def test_cfl_nested_tiers_match_c_oracle(coracle):
    d = configs.config2()[0]
    lv = _level(d, 0.9)
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, 6)
    c = configs.CONFIG2_PROBLEM
    pb = problem(d.dt, d.substeps, 1, final_time=d.final_time, cells=c["cells"], ic=c["ic"], box=c["qoi_box"],
                 domain=c["domain"], qoi_mean=True, tiers=d.tiers, cfl_safety=0.9)
    rc, _, oq, _, _ = coracle.eval_pairs(MeshArrays(*configs.build_mesh(d).arrays()), pb, None, None, 0, 0, 0, 6)
    assert rc == 0
    assert per_sample_rel(qf, oq) < QOI_RTOL


@pytest.mark.parametrize("kind", ["lts", "lf"])
def test_cfl_per_sample_steps_match_c_oracle(coracle, kind):
    """The device's per-sample (snapped) dt and step count against the C
    restatement of stable_dt (itself pinned to the reference above)."""
    d = configs.config0() if kind == "lts" else configs.config0_leapfrog()
    lv = _level(d, 0.9)
    dt, steps = wavemc.level_cfl(lv, 0, 0, 0, 70)
    ma = MeshArrays(*configs.build_mesh(d).arrays())
    pb = problem(d.dt, d.substeps, 1 if kind == "lts" else 0, cfl_safety=0.9)
    for i in (0, 1, 2, 33, 69):
        rc, odt, _ = coracle.stable_dt(ma, pb, coracle.draw_cells(0, 0, i))
        n = int(np.ceil(1.0 / odt - 1e-12))
        assert rc == 0 and steps[i] == n and abs(dt[i] - 1.0 / n) <= 1e-15, (i, steps[i], n)
