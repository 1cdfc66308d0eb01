"""Pin the C restatement (oracle/wmc_oracle.c) against golden vectors that the
UNMODIFIED reference produced (oracle/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle_py import MeshArrays, problem
from paper_2106_11117_b200 import configs


def test_rng_words_match_reference(golden, coracle):
    g = golden("rng.json")
    for case in g["words"]:
        words = coracle.stream_words(case["seed"], case["level"], case["index"], len(case["words"]))
        assert [hex(w) for w in words] == case["words"]
    # the survey's published probe values
    assert coracle.stream_words(0, 0, 0, 3) == [0x8b5ecfa548c96ac0, 0xc6b8327c8ac2b7d4, 0xa1414b2ed705eaec]


def test_rng_uniform_bit_identical(golden, coracle):
    for case in golden("rng.json")["uniform"]:
        got = coracle.draw_cells(case["seed"], case["level"], case["index"], len(case["values"]), case["lo"],
                                 case["hi"])
        assert got.tolist() == case["values"]  # bit-identical


def test_chebyshev_constants_match_reference(golden, coracle):
    for case in golden("chebyshev.json"):
        d, o, bi, bh = coracle.chebyshev(case["p"], case["nu"])
        assert d == case["delta"] and o == case["omega"]
        assert bi == case["beta_int"] and bh == case["beta_half"]


def test_chebyshev_rejects_bad_arguments(coracle):
    with pytest.raises(ValueError):
        coracle.chebyshev(0, 0.01)
    with pytest.raises(ValueError):
        coracle.chebyshev(4, 1.5)


@pytest.fixture(scope="module")
def config0_mesh():
    m = configs.build_mesh(configs.config0())
    return MeshArrays(*m.arrays())


def test_level_data_matches_reference(golden, coracle, config0_mesh):
    g = golden("config0_level.json")
    d = configs.config0()
    z0, mass, w = coracle.level_data(config0_mesh, problem(d.dt, d.substeps))
    np.testing.assert_allclose(z0, g["z0"], rtol=1e-14, atol=1e-300)
    np.testing.assert_allclose(mass, g["mass"], rtol=1e-14)
    np.testing.assert_allclose(w, g["qoi_w"], rtol=1e-14, atol=0)


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def test_config0_lts_samples_match_reference(golden, coracle, config0_mesh):
    g = golden("config0_samples.json")["lts"]
    pb = problem(g["dt"], g["p"], 1, nu=g["nu"])
    n = 8
    rc, dq, qf, _, _ = coracle.eval_pairs(config0_mesh, pb, None, None, 0, g["stream_level"], g["first"], n)
    assert rc == 0
    assert _rel(qf, g["q"][:n]) < 1e-12
    assert np.array_equal(dq, qf)


def test_config0_leapfrog_samples_match_reference(golden, coracle, config0_mesh):
    g = golden("config0_samples.json")["lf"]
    pb = problem(g["dt"], 1, 0)
    rc, dq, qf, _, _ = coracle.eval_pairs(config0_mesh, pb, None, None, 0, 0, 0, 4)
    assert rc == 0
    assert _rel(qf, g["q"][:4]) < 1e-12


def test_config0_nu0_offset_stream_matches_reference(golden, coracle, config0_mesh):
    g = golden("config0_samples.json")["lts_nu0"]
    pb = problem(g["dt"], g["p"], 1, nu=g["nu"])
    rc, _, qf, _, _ = coracle.eval_pairs(config0_mesh, pb, None, None, 0, g["stream_level"], g["first"], 4)
    assert rc == 0
    assert _rel(qf, g["q"][:4]) < 1e-12


def test_moments_fold_matches_reference(golden, coracle):
    lv = golden("config0_moments.json")["levels"][0]
    m = coracle.moments(np.array(lv["dq"]), np.array(lv["q"]))
    assert m["n"] == lv["N"]
    for k in ("sum_dq", "sum_dq2", "sum_q", "sum_q2", "variance", "mc_variance"):
        assert m[k] == pytest.approx(lv[k], rel=1e-14), k


def test_config1_level1_pair_matches_reference(golden, coracle):
    """Coupled pair (same draw on level 1 and level 0), reference sample_delta_q."""
    c1 = configs.config1()
    fine = MeshArrays(*configs.build_mesh(c1[1]).arrays())
    coarse = MeshArrays(*configs.build_mesh(c1[0]).arrays())
    lv = golden("config1_pairs.json")["levels"][1]
    rc, dq, qf, _, _ = coracle.eval_pairs(fine, problem(c1[1].dt, c1[1].substeps), coarse,
                                          problem(c1[0].dt, c1[0].substeps), 0, 1, 0, 2)
    assert rc == 0
    assert _rel(qf, lv["q"][:2]) < 1e-12
    assert np.max(np.abs(dq - lv["dq"][:2])) < 1e-12 * np.max(np.abs(qf))


def test_instability_reported_with_step(coracle, config0_mesh):
    """A coarse dt far above the CFL bound trips check_finite (integrators.cpp:12-18)."""
    pb = problem(0.2, 1, 0, final_time=20.0)  # leapfrog at dt = 0.2 on h_min = 1/128
    rc, q, step, _ = coracle.solve(config0_mesh, pb, np.ones(16))
    assert rc == 3 and step > 1


def test_kl_table_is_a_truncated_expansion():
    from paper_2106_11117_b200 import wavemc
    kl = configs.KL_FIELD
    table, lam = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
    assert table.shape == (kl["cells"][0] * kl["cells"][1], kl["modes"])
    assert np.all(np.diff(lam) <= 1e-15) and lam[0] < 1.0 and 0.3 < lam.sum() < 1.0
    # per-cell variance of g = sigma^2 sum_m lambda_m phi_m(x)^2 <= sigma^2
    var = np.sum(table ** 2, axis=1)
    assert np.all(var > 0) and np.all(var <= kl["sigma"] ** 2)


def test_config4_kl_pairs_match_reference(golden, coracle):
    """Config 4 (log-normal KL coefficient): the C restatement against the
    reference solver on the same cell coefficients."""
    from paper_2106_11117_b200 import wavemc
    kl = configs.KL_FIELD
    table, _ = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
    g = golden("config4_pairs.json")["levels"]
    c1 = configs.config1()
    fine = MeshArrays(*configs.build_mesh(c1[1]).arrays())
    coarse = MeshArrays(*configs.build_mesh(c1[0]).arrays())
    pf = problem(c1[1].dt, c1[1].substeps, cells=kl["cells"], kl_table=table)
    pc = problem(c1[0].dt, c1[0].substeps, cells=kl["cells"], kl_table=table)
    rc, dq, qf, _, _ = coracle.eval_pairs(fine, pf, coarse, pc, 0, 1, 0, 2)
    assert rc == 0
    assert _rel(qf, g[1]["q"][:2]) < 1e-12
    assert np.max(np.abs(dq - g[1]["dq"][:2])) < 1e-12 * np.max(np.abs(qf))


def test_cfl_per_sample_dt_matches_reference(golden, coracle, config0_mesh):
    """Per-sample CFL step (reference stable_dt, src/experiments.cpp:30-43, over
    max_eigenvalue / coarse_max_eigenvalue, src/fem.cpp:132-189)."""
    g = golden("cfl_samples.json")
    d = configs.config0()
    pb = problem(d.dt, d.substeps, 1, cfl_safety=g["safety"])
    rc, _, qf, _, _ = coracle.eval_pairs(config0_mesh, pb, None, None, 0, 0, 0, len(g["config0_lts"]["q"]))
    assert rc == 0 and _rel(qf, g["config0_lts"]["q"]) < 1e-12
    pb = problem(d.dt, 1, 0, cfl_safety=g["safety"])
    rc, _, qf, _, _ = coracle.eval_pairs(config0_mesh, pb, None, None, 0, 0, 0, len(g["config0_lf"]["q"]))
    assert rc == 0 and _rel(qf, g["config0_lf"]["q"]) < 1e-12
    # the step really is per sample and near the stability bound
    rc, dt0, it0 = coracle.stable_dt(config0_mesh, problem(d.dt, d.substeps, 1, cfl_safety=0.9),
                                     coracle.draw_cells(0, 0, 0))
    rc, dt1, it1 = coracle.stable_dt(config0_mesh, problem(d.dt, d.substeps, 1, cfl_safety=0.9),
                                     coracle.draw_cells(0, 0, 1))
    assert rc == 0 and dt0 != dt1 and 2 * d.dt < dt0 < 4 * d.dt and min(it0) >= 3


def test_cfl_pairs_match_reference(golden, coracle):
    g = golden("cfl_samples.json")
    c1 = configs.config1()
    fine = MeshArrays(*configs.build_mesh(c1[1]).arrays())
    coarse = MeshArrays(*configs.build_mesh(c1[0]).arrays())
    lv = g["config1_pairs"]["levels"][1]
    rc, dq, qf, _, _ = coracle.eval_pairs(fine, problem(c1[1].dt, c1[1].substeps, cfl_safety=g["safety"]), coarse,
                                          problem(c1[0].dt, c1[0].substeps, cfl_safety=g["safety"]), 0, 1, 0, lv["N"])
    assert rc == 0
    assert _rel(qf, lv["q"]) < 1e-12
    assert np.max(np.abs(dq - lv["dq"])) < 1e-12 * np.max(np.abs(qf))
