"""Parity of the CUDA path (through the C ABI) with the reference: golden
vectors from the unmodified reference library and the C restatement as the
checker.  Tolerances (BASELINE north_star): per-sample QoI within 1e-10
relative, per-level means and variances within 1e-9 relative."""
import numpy as np
import pytest

from oracle_py import MeshArrays, problem
from paper_2106_11117_b200 import configs, wavemc
from paper_2106_11117_b200._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING

pytestmark = pytest.mark.gpu

QOI_RTOL = 1e-10
MOMENT_RTOL = 1e-9


def rel_err(got, ref, scale=None):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    scale = np.max(np.abs(ref)) if scale is None else scale
    return float(np.max(np.abs(got - ref)) / scale)


def per_sample_rel(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


@pytest.fixture(scope="module")
def level0():
    return configs.build_level(configs.config0())


@pytest.fixture(scope="module")
def mesh0_arrays():
    return MeshArrays(*configs.build_mesh(configs.config0()).arrays())


def test_draw_cells_bit_identical_to_reference(golden):
    for case in golden("rng.json")["uniform"]:
        got = wavemc.draw_cells(case["seed"], case["level"], case["index"], 1, len(case["values"]), case["lo"],
                                case["hi"])
        assert got[0].tolist() == case["values"]


def test_draw_cells_match_c_oracle_many(coracle):
    got = wavemc.draw_cells(7, 3, 10**6, 300)
    for i in (0, 1, 63, 64, 299):
        assert got[i].tolist() == coracle.draw_cells(7, 3, 10**6 + i).tolist()


def test_level_info_matches_reference_counts(golden, level0):
    hdr = golden("config0_samples.json")["lts"]["header"]
    assert level0.info["n"] == int(hdr["n"])
    assert level0.info["n_r"] == int(hdr["n_r"])
    assert level0.info["n_steps"] == int(hdr["n_steps"])
    assert level0.info["dof_updates_per_solve"] == pytest.approx(float(hdr["dof_updates_per_solve"]))


def test_config0_lts_matches_reference(golden, level0):
    g = golden("config0_samples.json")["lts"]
    dq, qf, cost = wavemc.eval_pairs(level0, None, 0, 0, 0, len(g["q"]))
    assert per_sample_rel(qf, g["q"]) < QOI_RTOL
    assert np.array_equal(dq, qf)
    assert cost["matvec_fine"] == len(g["q"]) * (level0.info["n_steps"] - 1) * 4


def test_config0_lts_nu0_offset_stream_matches_reference(golden):
    g = golden("config0_samples.json")["lts_nu0"]
    d = configs.config0()
    lv = wavemc.Level(configs.build_mesh(d), wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, nu=0.0))
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, g["stream_level"], g["first"], len(g["q"]))
    assert per_sample_rel(qf, g["q"]) < QOI_RTOL


def test_config0_leapfrog_matches_reference(golden):
    g = golden("config0_samples.json")["lf"]
    lv = configs.build_level(configs.config0_leapfrog())
    _, qf, cost = wavemc.eval_pairs(lv, None, 0, 0, 0, len(g["q"]))
    assert per_sample_rel(qf, g["q"]) < QOI_RTOL
    assert cost["matvec_full"] == len(g["q"]) * lv.info["n_steps"]


def test_config0_matches_c_oracle(coracle, level0, mesh0_arrays):
    d = configs.config0()
    n = 48
    _, qf, _ = wavemc.eval_pairs(level0, None, 0, 0, 500, n)
    rc, _, ref, _, _ = coracle.eval_pairs(mesh0_arrays, problem(d.dt, d.substeps), None, None, 0, 0, 500, n)
    assert rc == 0
    assert per_sample_rel(qf, ref) < QOI_RTOL


def test_config1_pairs_every_level_match_reference(golden):
    levels = [configs.build_level(d) for d in configs.config1()]
    for lv in golden("config1_pairs.json")["levels"]:
        l, n = lv["level"], lv["N"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        # dQ is a difference of O(|Q|) numbers: hold it to the QoI budget of Q
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l


def test_fixed_mlmc_moments_match_reference(golden, level0):
    lv = golden("config0_moments.json")["levels"][0]
    st = wavemc.run_mlmc_fixed([level0], [lv["N"]], seed=0)[0]
    assert st["n_samples"] == lv["N"]
    for k in ("sum_dq", "sum_q", "variance", "mc_variance", "mean_dq", "sum_dq2", "sum_q2"):
        assert st[k] == pytest.approx(lv[k], rel=MOMENT_RTOL), k


def test_batching_and_offsets_are_bitwise_invariant():
    d = configs.config0()
    small = configs.build_level(d, batch=64)
    big = configs.build_level(d, batch=1024)
    _, a, _ = wavemc.eval_pairs(small, None, 0, 0, 0, 200)
    _, b, _ = wavemc.eval_pairs(big, None, 0, 0, 0, 200)
    _, c, _ = wavemc.eval_pairs(big, None, 0, 0, 37, 100)
    assert np.array_equal(a, b)
    assert np.array_equal(a[37:137], c)


def test_repeat_runs_are_bitwise_identical(level0):
    _, a, _ = wavemc.eval_pairs(level0, None, 3, 1, 0, 300)
    _, b, _ = wavemc.eval_pairs(level0, None, 3, 1, 0, 300)
    assert np.array_equal(a, b)


def test_lts_p1_nu0_equals_leapfrog():
    """reference tests/test_integrators.cpp:217-236 on the P1 mesh."""
    d = configs.config0()
    dt = 0.2 / 128
    lts = wavemc.Level(configs.build_mesh(d), wavemc.LevelSpec(dt=dt, substeps=1, nu=0.0))
    lf = wavemc.Level(configs.build_mesh(d), wavemc.LevelSpec(dt=dt, integrator=WMC_LEAPFROG))
    _, a, _ = wavemc.eval_pairs(lts, None, 0, 0, 0, 64)
    _, b, _ = wavemc.eval_pairs(lf, None, 0, 0, 0, 64)
    assert rel_err(a, b) < 1e-12


def test_empty_selector_equals_leapfrog():
    """reference tests/test_integrators.cpp:238-265: P empty -> LTS == LF."""
    mesh = wavemc.Mesh.build_square(32, 4, small_factor=0.0)
    _, _, fine, _ = mesh.arrays()
    assert fine.sum() == 0
    dt = 0.2 / 128
    lts = wavemc.Level(mesh, wavemc.LevelSpec(dt=dt, substeps=16, nu=0.01))
    assert lts.info["n_r"] == 0
    lf = wavemc.Level(mesh, wavemc.LevelSpec(dt=dt, integrator=WMC_LEAPFROG))
    _, a, ca = wavemc.eval_pairs(lts, None, 0, 0, 0, 64)
    _, b, _ = wavemc.eval_pairs(lf, None, 0, 0, 0, 64)
    assert rel_err(a, b) < 1e-11
    assert ca["matvec_fine"] == 64 * (lts.info["n_steps"] - 1) * 16


def test_instability_raises_numerical_error_with_step(coracle, mesh0_arrays):
    lv = wavemc.Level(configs.build_mesh(configs.config0()),
                      wavemc.LevelSpec(dt=0.2, final_time=20.0, integrator=WMC_LEAPFROG))
    with pytest.raises(wavemc.NumericalError) as ei:
        wavemc.eval_pairs(lv, None, 0, 0, 5, 3)
    assert ei.value.sample == 5
    rc, _, step, _ = coracle.solve(mesh0_arrays, problem(0.2, 1, 0, final_time=20.0),
                                   coracle.draw_cells(0, 0, 5))
    assert rc == 3 and ei.value.step == step


def test_fused_solve_reports_instability_like_the_step_kernels(monkeypatch):
    """An unstable LF-LTS level (coarse step far above its CFL bound) through
    the fused lattice solve reports the same first failing sample and step as
    the per-step kernels (check_finite, src/integrators.cpp:12-18)."""
    d = configs.config1()[0]
    spec = configs.level_spec(d)
    spec.dt = 4.0 * spec.dt
    m = configs.build_mesh(d)
    fused = wavemc.Level(m, spec)
    monkeypatch.setenv("WMC_FUSED", "0")
    plain = wavemc.Level(m, spec)
    monkeypatch.delenv("WMC_FUSED")
    assert fused.info["fused"] == 1 and plain.info["fused"] == 0
    errs = []
    for lv in (fused, plain):
        with pytest.raises(wavemc.NumericalError) as ei:
            wavemc.eval_pairs(lv, None, 0, 0, 3, 40)
        errs.append((ei.value.sample, ei.value.step))
    assert errs[0] == errs[1] and errs[0][0] == 3 and errs[0][1] > 1


def test_config_errors_are_reported():
    with pytest.raises(wavemc.ConfigError):
        wavemc.Level(configs.build_mesh(configs.config0()), wavemc.LevelSpec(dt=0.01, nu=2.0))
    with pytest.raises(wavemc.ConfigError):
        wavemc.Level(configs.build_mesh(configs.config0()), wavemc.LevelSpec(dt=-1.0))


def test_lattice_and_generic_substep_kernels_agree():
    """The structured refined-square kernel against the generic SELL kernel on
    the same mesh (a mesh passed as arrays carries no lattice block)."""
    for d in (configs.config0(), configs.config1()[0], configs.config1()[2]):
        m = configs.build_mesh(d)
        lat = wavemc.Level(m, configs.level_spec(d))
        gen = wavemc.Level(wavemc.Mesh.from_arrays(*m.arrays()), configs.level_spec(d))
        assert lat.info["lattice"] == 1 and gen.info["lattice"] == 0
        _, a, _ = wavemc.eval_pairs(lat, None, 0, 1, 0, 40)
        _, b, _ = wavemc.eval_pairs(gen, None, 0, 1, 0, 40)
        assert per_sample_rel(a, b) < QOI_RTOL


def test_concurrent_levels_use_separate_workspaces():
    """Pairs of adjacent levels issued back to back on their own streams share
    the middle level (fine of one pair, coarse of the next)."""
    import torch
    levels = [configs.build_level(d, batch=256) for d in configs.config1()[:3]]
    n = 300
    ref = [wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n) for l in range(3)]
    d_dq = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    d_qf = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
    for l in range(3):
        wavemc.eval_pairs_device(levels[l], levels[l - 1] if l else None, 0, l, 0, n, d_dq[l].data_ptr(),
                                 d_qf[l].data_ptr())
    for lv in levels:
        wavemc.synchronize(lv)
    for l in range(3):
        assert np.array_equal(d_dq[l].cpu().numpy(), ref[l][0]), l
        assert np.array_equal(d_qf[l].cpu().numpy(), ref[l][1]), l


def test_config1_level0_full_batch_spot_checks(coracle):
    """Full-size run (65536 samples of config 1 level 0): spot indices against
    the C oracle, and the batch result is independent of the index range."""
    d = configs.config1()[0]
    lv = configs.build_level(d)
    n = 65536
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, n)
    assert np.all(np.isfinite(qf))
    mesh = MeshArrays(*configs.build_mesh(d).arrays())
    for i in (0, 4095, 4096, 40000, n - 1):
        rc, _, ref, _, _ = coracle.eval_pairs(mesh, problem(d.dt, d.substeps), None, None, 0, 0, i, 1)
        assert rc == 0
        assert abs(qf[i] - ref[0]) / abs(ref[0]) < QOI_RTOL, i
    _, tail, _ = wavemc.eval_pairs(lv, None, 0, 0, n - 100, 100)
    assert np.array_equal(tail, qf[-100:])


def test_adaptive_mlmc_matches_reference_run_mlmc(golden):
    """wmc_run_mlmc against the reference's own run_mlmc (src/mlmc.cpp:165-233)
    on the config-1 hierarchy: same sample counts per level, estimates within
    the moment tolerance."""
    g = golden("config1_adaptive.json")
    levels = [configs.build_level(d) for d in configs.config1()]
    res = wavemc.run_mlmc(levels, g["model_cost"], wavemc.MlmcConfig(eps=g["eps"]))
    assert res.converged == g["converged"]
    assert res.levels_used + 1 == len(g["levels"])
    for got, want in zip(res.levels, g["levels"]):
        assert got["n_samples"] == want["N"]
        assert got["variance"] == pytest.approx(want["variance"], rel=MOMENT_RTOL)
    assert res.estimate == pytest.approx(g["estimate"], rel=MOMENT_RTOL)
    assert res.total_variance == pytest.approx(g["total_variance"], rel=MOMENT_RTOL)
    assert res.bias == pytest.approx(g["bias"], rel=MOMENT_RTOL)


@pytest.mark.parametrize("lvl", [0, 1, 2])
def test_fused_lattice_solve_matches_the_step_kernels(lvl, monkeypatch):
    """The fused lattice solve (whole solves on chip, one launch per batch)
    against the per-step sweep / lattice substep / R update kernels on
    config-1 level meshes (fused on levels 0 and 1; level 2 is forced onto
    the global-history layout): the same operator, lattice rows' A z_n from
    the substep stencil instead of the sweep descriptors, so agreement at
    rounding level."""
    defs = configs.config1()
    if lvl == 2:
        monkeypatch.setenv("WMC_FUSED_ZP_GLOBAL", "1")
    fused = [configs.build_level(d) for d in defs[max(lvl - 1, 0):lvl + 1]]
    monkeypatch.delenv("WMC_FUSED_ZP_GLOBAL", raising=False)
    monkeypatch.setenv("WMC_FUSED", "0")
    plain = [configs.build_level(d) for d in defs[max(lvl - 1, 0):lvl + 1]]
    monkeypatch.delenv("WMC_FUSED")
    assert fused[-1].info["fused"] in (1, 2) and plain[-1].info["fused"] == 0
    assert fused[-1].info["substep_path"] == plain[-1].info["substep_path"] == 1
    pair = (lambda lv: (lv[-1], lv[0] if lvl else None))
    n = 300 if lvl < 2 else 90
    dq_f, qf_f, _ = wavemc.eval_pairs(*pair(fused), 0, lvl, 5, n)
    dq_p, qf_p, _ = wavemc.eval_pairs(*pair(plain), 0, lvl, 5, n)
    assert per_sample_rel(qf_f, qf_p) < 1e-12
    assert np.max(np.abs(dq_f - dq_p) / np.abs(qf_p)) < 1e-12


@pytest.mark.parametrize("lvl,form", [(0, "2"), (1, "2"), (1, "1")])
def test_fused_solve_tensor_memory_is_bitwise_the_shared_memory_form(lvl, form, monkeypatch):
    """The fused solve keeps each thread's generic SELL weights / columns
    (form 2, default) and optionally its lattice nodes' d_{m-1} (form 1) in
    tensor memory (tcgen05.ld / st) instead of shared memory: the same
    products in the same order, so the same bits (coupled pairs, level-1
    pairs include a level-0 coarse solve)."""
    defs = configs.config1()
    monkeypatch.setenv("WMC_FUSED_TMEM", form)
    a = [configs.build_level(d) for d in defs[max(lvl - 1, 0):lvl + 1]]
    monkeypatch.setenv("WMC_FUSED_TMEM", "0")
    b = [configs.build_level(d) for d in defs[max(lvl - 1, 0):lvl + 1]]
    monkeypatch.delenv("WMC_FUSED_TMEM")
    assert a[-1].info["fused"] == b[-1].info["fused"] == 1
    pair = (lambda lv: (lv[-1], lv[0] if lvl else None))
    dq_a, qa, _ = wavemc.eval_pairs(*pair(a), 0, lvl, 3, 400)
    dq_b, qb, _ = wavemc.eval_pairs(*pair(b), 0, lvl, 3, 400)
    assert np.array_equal(qa, qb) and np.array_equal(dq_a, dq_b)


def test_fused_lattice_solve_with_global_history(monkeypatch):
    """z_{n-1} in the per-sample global buffer instead of shared memory (the
    layout levels with larger n take) gives the same bits."""
    d = configs.config1()[1]
    a = configs.build_level(d)
    monkeypatch.setenv("WMC_FUSED_ZP_GLOBAL", "1")
    b = configs.build_level(d)
    monkeypatch.delenv("WMC_FUSED_ZP_GLOBAL")
    assert a.info["fused"] == 1 and b.info["fused"] == 2
    _, qa, _ = wavemc.eval_pairs(a, None, 0, 1, 0, 200)
    _, qb, _ = wavemc.eval_pairs(b, None, 0, 1, 0, 200)
    assert np.array_equal(qa, qb)


@pytest.mark.parametrize("path", ["global", "onchip"])
def test_substep_paths_agree(path, monkeypatch):
    """The HBM-resident and the generic on-chip substep kernels against the
    lattice kernel (and, through it, the reference) on config-0 and config-1
    level meshes."""
    for d in (configs.config0(), configs.config1()[1]):
        ref = configs.build_level(d)
        monkeypatch.setenv("WMC_SUBSTEP_PATH", path)
        alt = configs.build_level(d)
        monkeypatch.delenv("WMC_SUBSTEP_PATH")
        assert ref.info["substep_path"] == 1
        assert alt.info["substep_path"] == {"global": 3, "onchip": 2}[path]
        _, a, _ = wavemc.eval_pairs(ref, None, 0, 2, 0, 70)
        _, b, _ = wavemc.eval_pairs(alt, None, 0, 2, 0, 70)
        assert per_sample_rel(b, a) < QOI_RTOL


def test_large_r_uses_the_hbm_path():
    """A refined square of 256 x 256 fine cells (|R| > 8192) cannot live in one
    SM: the level falls back to the HBM-resident substep kernel and still
    matches the C oracle."""
    m = wavemc.Mesh.build_square(32, 64)
    lv = wavemc.Level(m, wavemc.LevelSpec(dt=0.2 / 32, substeps=64, final_time=0.05))
    assert lv.info["n_r"] > 8192 and lv.info["substep_path"] == 3
    _, q, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, 3)
    import oracle_py
    orc = oracle_py.COracle()
    rc, _, ref, _, _ = orc.eval_pairs(oracle_py.MeshArrays(*m.arrays()),
                                     oracle_py.problem(0.2 / 32, 64, final_time=0.05), None, None, 0, 0, 0, 3)
    assert rc == 0
    assert per_sample_rel(q, ref) < QOI_RTOL


def _kl_levels(n=5):
    return [configs.build_level(d, kl=True) for d in configs.config4()[:n]]


def test_kl_draw_matches_c_oracle(coracle):
    kl = configs.KL_FIELD
    table, _ = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
    lv = _kl_levels(1)[0]
    got = wavemc.level_draw(lv, 0, 2, 777, 130)
    for i in (0, 1, 64, 129):
        ref = coracle.draw_kl(0, 2, 777 + i, table)
        assert np.max(np.abs(got[i] - ref) / ref) < 1e-14


def test_config4_pairs_match_reference(golden):
    levels = _kl_levels(3)
    for lv in golden("config4_pairs.json")["levels"]:
        l, n = lv["level"], lv["N"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l


@pytest.mark.parametrize("target", ["baseline", "tight"])
def test_config4_adaptive_mlmc_matches_reference(golden, target):
    """Config 4 (log-normal KL on the 32 x 32 cell grid): the adaptive driver
    against the reference's run_mlmc at the BASELINE target 1e-3 (met by the
    warm-up) and at 1.5e-4 (more samples and levels)."""
    g0 = golden("config4_adaptive.json")
    g = g0 if target == "baseline" else g0["tight"]
    assert tuple(g0["cells"]) == tuple(configs.KL_FIELD["cells"])
    res = wavemc.run_mlmc(_kl_levels(), g0["model_cost"], wavemc.MlmcConfig(eps=g["eps"]))
    assert res.converged == g["converged"]
    assert [lv["n_samples"] for lv in res.levels] == [lv["N"] for lv in g["levels"]]
    assert res.estimate == pytest.approx(g["estimate"], rel=MOMENT_RTOL)
    for got, want in zip(res.levels, g["levels"]):
        assert got["variance"] == pytest.approx(want["variance"], rel=MOMENT_RTOL)


def _kl_element_levels(n=5):
    return [configs.build_level(d, kl="element") for d in configs.config4()[:n]]


def test_config4_element_field_pairs_match_reference(golden):
    """Config 4 with the KL field at every triangle's centroid -- the rule of
    the reference's assemble (src/fem.cpp:103-104), which calls
    speed2(x, y) = exp(g(x, y)) itself on its side: one draw per pair, each
    level on its own elements."""
    levels = _kl_element_levels(3)
    assert all(lv.info["lattice"] == 0 for lv in levels)  # one coefficient per triangle: generic kernels
    for lv in golden("config4_element.json")["pairs"]["levels"]:
        l, n = lv["level"], lv["N"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l


def test_config4_element_field_pairs_on_all_levels(golden):
    """One coupled pair per level, levels 3-4 included (41 k / 136 k triangles:
    cells beside 16-bit columns, and the per-entry cell arrays of the sweep
    and of the HBM-resident substeps)."""
    levels = _kl_element_levels(5)
    for lv in golden("config4_element.json")["pairs_all_levels"]["levels"]:
        l, n = lv["level"], lv["N"]
        dq, qf, _ = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, n)
        assert per_sample_rel(qf, lv["q"]) < QOI_RTOL, l
        assert np.max(np.abs(dq - lv["dq"]) / np.abs(lv["q"])) < 2 * QOI_RTOL, l


@pytest.mark.parametrize("target", ["adaptive", "tight"])
def test_config4_element_field_adaptive_mlmc_matches_reference(golden, target):
    g0 = golden("config4_element.json")
    g = g0[target]
    res = wavemc.run_mlmc(_kl_element_levels(), g0["model_cost"], wavemc.MlmcConfig(eps=g["eps"]))
    assert res.converged == g["converged"]
    assert [lv["n_samples"] for lv in res.levels] == [lv["N"] for lv in g["levels"]]
    assert res.estimate == pytest.approx(g["estimate"], rel=MOMENT_RTOL)
    for got, want in zip(res.levels, g["levels"]):
        assert got["variance"] == pytest.approx(want["variance"], rel=MOMENT_RTOL)


def test_adaptive_driver_evaluate_ahead_is_invisible(monkeypatch):
    """The driver's evaluate-ahead cache (64-lane granules, next level's
    warm-up beside the current wave) folds exactly the reference's samples:
    same N_l, bitwise the same estimate and sums as plain waves."""
    levels = [configs.build_level(d) for d in configs.config1()[:4]]
    costs = [lv.info["dof_updates_per_solve"] for lv in levels]
    cfg = wavemc.MlmcConfig(eps=3e-4)
    a = wavemc.run_mlmc(levels, costs, cfg)
    monkeypatch.setenv("WMC_MLMC_NO_AHEAD", "1")
    b = wavemc.run_mlmc(levels, costs, cfg)
    assert [s["n_samples"] for s in a.levels] == [s["n_samples"] for s in b.levels]
    assert a.estimate == b.estimate and a.rmse == b.rmse
    for x, y in zip(a.levels, b.levels):
        assert x["sum_dq"] == y["sum_dq"] and x["sum_q2"] == y["sum_q2"]


@pytest.mark.parametrize("case", ["lattice", "global", "tiers"])
def test_wide_sweep_is_bitwise_the_two_sample_sweep(case, monkeypatch):
    """The 256-bit step sweep (four samples per lane, default for fixed dt
    and batches of 128k samples) against the 16-byte sweep_rows_kernel: the
    same per-sample products and sums, so the same bits -- g stashed
    sample-major (lattice substeps, config-1 level 3), node-major (the
    HBM-resident substep path) and on the nested-tier path (config 2)."""
    if case == "tiers":
        d = configs.config2()[1]
    else:
        d = configs.config1()[3 if case == "lattice" else 1]
    if case == "global":
        monkeypatch.setenv("WMC_SUBSTEP_PATH", "global")
        monkeypatch.setenv("WMC_FUSED", "0")
    a = configs.build_level(d)
    monkeypatch.setenv("WMC_SWEEP_WIDE", "0")
    b = configs.build_level(d)
    _, qa, _ = wavemc.eval_pairs(a, None, 0, 1, 0, 256)
    _, qb, _ = wavemc.eval_pairs(b, None, 0, 1, 0, 256)
    assert np.all(np.isfinite(qa))
    assert np.array_equal(qa, qb)


@pytest.mark.parametrize("n_coarse,ratio", [(16, 4), (32, 8)])
def test_fused_solve_with_short_strips_matches_the_step_kernels(n_coarse, ratio, monkeypatch):
    """Refined squares whose lattice runs cut into strips shorter than K - 1
    (h_min = 1/64: runs of 3 rows) or into K / K - 1 strips (h_min = 1/256:
    runs of 31) take the fused solve's general and compiled-out short-strip
    forms; both against the per-step kernels at rounding level."""
    d = configs.LevelDef(n_coarse, ratio, 0.2 / n_coarse, ratio, configs.config1()[0].integrator, final_time=0.25)
    fused = configs.build_level(d)
    monkeypatch.setenv("WMC_FUSED", "0")
    plain = configs.build_level(d)
    monkeypatch.delenv("WMC_FUSED")
    assert fused.info["fused"] == 1 and plain.info["fused"] == 0
    _, qf, _ = wavemc.eval_pairs(fused, None, 0, 0, 0, 300)
    _, qp, _ = wavemc.eval_pairs(plain, None, 0, 0, 0, 300)
    assert np.all(np.isfinite(qf))
    assert per_sample_rel(qf, qp) < 1e-12
