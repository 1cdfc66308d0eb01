"""Config 2 (graded L-shape, nested tiers) on the CPU side.

The reference has neither the L-shaped graded mesh with fine flags nor a
nested (multi-tier) LTS, so the nested scheme is "parity unpinned by the
reference".  What the reference can pin, it pins here:
  * geometry, Dirichlet boundary, coefficient grid, IC and QoI of config 2,
    through two solvers it has on the same mesh: single-tier LF-LTS with
    P = P_1, p = 8 and global leap-frog at dt / 8 (golden vectors from the
    unmodified reference, oracle/make_golden.py --only-config2);
  * the nested recursion by reduction: with every vertex in every tier and
    nu = 0 it is leap-frog at dt / p^tiers on a consistent history (the
    reference's own check for one tier, tests/test_integrators.cpp:267-306),
    and with empty deeper tiers it is the single-tier scheme.
"""
import numpy as np
import pytest

from oracle_py import MeshArrays, problem
from paper_2106_11117_b200 import configs, wavemc


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def _c2_problem(d, substeps=None, kind=1, tiers=None, dt=None, nu=0.01):
    c = configs.CONFIG2_PROBLEM
    return problem(d.dt if dt is None else dt, d.substeps if substeps is None else substeps, kind,
                   final_time=d.final_time, nu=nu, cells=c["cells"], ic=c["ic"], box=c["qoi_box"],
                   domain=c["domain"], qoi_mean=True, tiers=d.tiers if tiers is None else tiers)


@pytest.fixture(scope="module")
def level0():
    d = configs.config2()[0]
    m = configs.build_mesh(d)
    return d, m, MeshArrays(*m.arrays())


def test_lshape_mesh_geometry_and_tiers(golden):
    g = golden("config2_reductions.json")["meshes"]
    for l, d in enumerate(configs.config2(3)):
        xy, tri, fine, bnd = configs.build_mesh(d).arrays()
        ref = g[f"config2_l{l}"]
        assert ref["conforming"] and ref["positive_areas"] and ref["euler"] == 1
        assert (len(xy), len(tri)) == (ref["n_vertices"], ref["n_triangles"])
        a = xy[tri]
        area = 0.5 * ((a[:, 1, 0] - a[:, 0, 0]) * (a[:, 2, 1] - a[:, 0, 1])
                      - (a[:, 2, 0] - a[:, 0, 0]) * (a[:, 1, 1] - a[:, 0, 1]))
        assert np.all(area > 0) and area.sum() == pytest.approx(3.0, rel=1e-14)
        # nothing in the removed quadrant
        c = a.mean(axis=1)
        assert not np.any((c[:, 0] > 0) & (c[:, 1] < 0))
        # all three tiers present, deepest tier at the corner, sizes h / 2^k
        assert set(np.unique(fine)) == {0, 1, 2, 3}
        near = np.hypot(c[:, 0], c[:, 1]) < 0.01
        assert np.all(fine[near] == 3)
        edge = np.max(np.hypot(*(a[:, 1] - a[:, 0]).T.reshape(2, -1)))
        assert edge <= np.sqrt(2) / d.n_coarse + 1e-12
        # boundary: the six sides of the L, including the re-entrant edges
        b = xy[bnd == 1]
        on = ((np.abs(np.abs(b[:, 0]) - 1) < 1e-14) | (np.abs(np.abs(b[:, 1]) - 1) < 1e-14)
              | ((np.abs(b[:, 0]) < 1e-14) & (b[:, 1] <= 0)) | ((np.abs(b[:, 1]) < 1e-14) & (b[:, 0] >= 0)))
        assert np.all(on)


def test_level_plan_nested_tiers():
    d = configs.config2()[1]
    info = wavemc.level_plan(configs.build_mesh(d), configs.level_spec(d))
    assert info["tiers"] == 3
    r = info["n_r_tier"]
    assert r[0] == info["n_r"] and r[0] > r[1] > r[2] > 0
    n, p, steps = info["n"], info["p"], info["n_steps"]
    assert steps == round(2.0 / d.dt)
    want = n + (steps - 1) * (n + (p - 1) * r[0] + (p * p - p) * r[1] + (p ** 3 - p * p) * r[2])
    assert info["dof_updates_per_solve"] == pytest.approx(want, rel=1e-15)


def test_nested_tiers_need_lts_with_substeps():
    d = configs.config2()[0]
    m = configs.build_mesh(d)
    spec = configs.level_spec(d)
    spec.substeps = 1
    with pytest.raises(wavemc.ConfigError):
        wavemc.level_plan(m, spec)


def test_single_tier_on_lshape_matches_reference(golden, coracle, level0):
    """Single-tier LF-LTS (P = P_1, p = 8) on the config-2 mesh and problem."""
    d, _, ma = level0
    g = golden("config2_reductions.json")["levels"][0]
    for key in ("lts_single_tier", "lts_single_tier_nu0"):
        c = g[key]
        pb = _c2_problem(d, substeps=c["p"], tiers=1, nu=c["nu"])
        rc, _, qf, _, _ = coracle.eval_pairs(ma, pb, None, None, 0, c["stream_level"], c["first"], len(c["q"]))
        assert rc == 0
        assert _rel(qf, c["q"]) < 1e-12, key


def test_leapfrog_on_lshape_matches_reference(golden, coracle, level0):
    d, _, ma = level0
    c = golden("config2_reductions.json")["levels"][0]["lf"]
    pb = _c2_problem(d, substeps=1, kind=0, tiers=1, dt=c["dt"])
    rc, _, qf, _, _ = coracle.eval_pairs(ma, pb, None, None, 0, 0, 0, len(c["q"]))
    assert rc == 0
    assert _rel(qf, c["q"]) < 1e-12


def test_nested_full_selection_is_leapfrog_at_finest_step(coracle):
    """Every vertex in every tier, nu = 0: the nested step from the pair
    (y_0, y_8) of a leap-frog trajectory at dt/8 reproduces y_16, y_24, ..."""
    d = configs.config2()[0]
    xy, tri, fine, bnd = configs.build_mesh(d).arrays()
    ma = MeshArrays(xy, tri, np.full_like(fine, 3), bnd)
    n = int((bnd == 0).sum())
    rng = np.random.default_rng(7)
    y0 = rng.standard_normal(n)
    y1 = y0 + 1e-3 * rng.standard_normal(n)
    cells = coracle.draw_cells(0, 0, 3, 64)
    dt = 0.05 / d.n_coarse
    lf = _c2_problem(d, substeps=1, kind=0, tiers=1, dt=dt / 8)
    traj = [y0, y1]
    zp, zc = y0.copy(), y1.copy()
    for _ in range(8 * 6):
        rc, zp, zc = coracle.steps(ma, lf, cells, zp, zc, 1)
        assert rc == 0
        traj.append(zc)
    nested = _c2_problem(d, substeps=2, tiers=3, dt=dt, nu=0.0)
    zp, zc = traj[0].copy(), traj[8].copy()
    for s in range(1, 6):
        rc, zp, zc = coracle.steps(ma, nested, cells, zp, zc, 1)
        assert rc == 0
        assert _rel(zc, traj[8 * (s + 1)]) < 1e-11


def test_nested_with_empty_deeper_tiers_is_single_tier(coracle, level0):
    d, _, ma = level0
    capped = MeshArrays(ma.xy, ma.tri, np.minimum(ma.fine, 1), ma.boundary)
    dt = 0.05 / d.n_coarse  # stable for the single tier at p = 2
    one = _c2_problem(d, substeps=2, tiers=1, dt=dt)
    three = _c2_problem(d, substeps=2, tiers=3, dt=dt)
    _, _, q1, _, _ = coracle.eval_pairs(capped, one, None, None, 0, 0, 0, 3)
    _, _, q3, _, _ = coracle.eval_pairs(capped, three, None, None, 0, 0, 0, 3)
    assert _rel(q3, q1) < 1e-12


def test_nested_tiers_stable_where_single_tier_is_not(coracle, level0):
    """p = 2 on P_1 alone cannot integrate the h/8 elements at dt = 0.2 h;
    three nested tiers of p = 2 can (the point of config 2)."""
    d, _, ma = level0
    rc1, _, _, _, _ = coracle.eval_pairs(ma, _c2_problem(d, tiers=1), None, None, 0, 0, 0, 4)
    rc3, _, q3, _, _ = coracle.eval_pairs(ma, _c2_problem(d), None, None, 0, 0, 0, 4)
    assert rc1 == 3 and rc3 == 0 and np.all(np.isfinite(q3))
    # and it agrees with the single-tier p = 8 solution to discretisation accuracy
    _, _, q8, _, _ = coracle.eval_pairs(ma, _c2_problem(d, substeps=8, tiers=1), None, None, 0, 0, 0, 4)
    assert _rel(q3, q8) < 5e-3
