"""Host-side checks that need no GPU: the C ABI library loads and exports
every symbol the public header declares, the mesh builder, and the level
tables (through the host-only wmc_level_plan)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2106_11117_b200 import _native, configs, wavemc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            with open(os.path.join(ROOT, "include", fn)) as f:
                text = f.read()
            names |= set(re.findall(r"^\s*[\w\s\*]*?\b(wmc_\w+)\s*\(", text, re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    declared = header_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    # and the Python binding covers them all
    assert declared == {n for n, _, _ in _native.SIGNATURES}


def edge_counts(tri):
    e = np.sort(np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]]), axis=1)
    _, counts = np.unique(e, axis=0, return_counts=True)
    return e, counts


@pytest.mark.parametrize("n_coarse,ratio", [(32, 4), (16, 32), (64, 8), (256, 2), (8, 1)])
def test_square_mesh_is_conforming_and_covers_the_square(n_coarse, ratio):
    m = wavemc.Mesh.build_square(n_coarse, ratio)
    xy, tri, fine, boundary = m.arrays()
    a, b, c = xy[tri[:, 0]], xy[tri[:, 1]], xy[tri[:, 2]]
    area = 0.5 * ((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    assert np.all(area > 0)
    assert area.sum() == pytest.approx(1.0, rel=1e-14)
    _, counts = edge_counts(tri)
    assert set(np.unique(counts)) <= {1, 2}  # conforming: interior edges shared by exactly two triangles
    nv, nt = len(xy), len(tri)
    ne = len(counts)
    assert nv - ne + nt == 1  # Euler characteristic of a disc
    on_edge = (xy[:, 0] == 0) | (xy[:, 1] == 0) | (xy[:, 0] == 1) | (xy[:, 1] == 1)
    assert np.array_equal(boundary.astype(bool), on_edge)
    # the refined square is a uniform lattice at h / ratio
    h_min = 1.0 / (n_coarse * ratio)
    inside = np.all((xy[tri].mean(axis=1) > 0.4375) & (xy[tri].mean(axis=1) < 0.5625), axis=1)
    if ratio > 1:
        assert np.allclose(np.abs(area[inside]), 0.5 * h_min * h_min)
        assert fine[inside].all()
    else:
        assert fine.sum() == 0


def test_mesh_matches_reference_checks(golden):
    g = golden("meshes.json")
    for name, d in [("config0", configs.config0())] + [(f"config1_l{l}", d) for l, d in enumerate(configs.config1())]:
        xy, tri, fine, _ = configs.build_mesh(d).arrays()
        assert len(xy) == g[name]["n_vertices"] and len(tri) == g[name]["n_triangles"]
        assert int(fine.sum()) == g[name]["n_fine"]
        assert g[name]["conforming"] and g[name]["positive_areas"] and g[name]["euler"] == 1


def test_level_plan_counts_match_reference(golden):
    hdr = golden("config0_samples.json")["lts"]["header"]
    d = configs.config0()
    info = wavemc.level_plan(configs.build_mesh(d), configs.level_spec(d))
    assert info["n"] == int(hdr["n"]) and info["n_r"] == int(hdr["n_r"]) and info["n_steps"] == int(hdr["n_steps"])
    assert info["dof_updates_per_solve"] == float(hdr["dof_updates_per_solve"])
    for lv in golden("config1_pairs.json")["levels"]:
        dd = configs.config1()[lv["level"]]
        info = wavemc.level_plan(configs.build_mesh(dd), configs.level_spec(dd))
        assert (info["n"], info["n_r"], info["n_steps"]) == (lv["n"], lv["n_r"], lv["n_steps"])


def test_level_plan_config_errors():
    m = configs.build_mesh(configs.config0())
    with pytest.raises(wavemc.ConfigError):
        wavemc.level_plan(m, wavemc.LevelSpec(dt=0.01, nu=1.5))
    with pytest.raises(wavemc.ConfigError):
        wavemc.level_plan(m, wavemc.LevelSpec(dt=0.0))
    with pytest.raises(wavemc.ConfigError):
        wavemc.level_plan(m, wavemc.LevelSpec(dt=0.01, substeps=0))
    with pytest.raises(wavemc.ConfigError):
        wavemc.level_plan(m, wavemc.LevelSpec(dt=0.01, integrator=7))
    with pytest.raises(wavemc.ConfigError):
        wavemc.Mesh.build_square(32, 3)  # ratio must be a power of two


def test_leapfrog_plan_has_no_substeps():
    d = configs.config0_leapfrog()
    info = wavemc.level_plan(configs.build_mesh(d), configs.level_spec(d))
    assert info["p"] == 1 and info["n_steps"] == 640
    assert info["dof_updates_per_solve"] == 640 * info["n"]


def test_mesh_round_trip_through_arrays():
    m = configs.build_mesh(configs.config0())
    xy, tri, fine, boundary = m.arrays()
    m2 = wavemc.Mesh.from_arrays(xy, tri, fine, boundary, 1 / 32, 1 / 128)
    xy2, tri2, fine2, b2 = m2.arrays()
    assert np.array_equal(xy, xy2) and np.array_equal(tri, tri2)
    assert np.array_equal(fine, fine2) and np.array_equal(boundary, b2)
    a = wavemc.level_plan(m, configs.level_spec(configs.config0()))
    b = wavemc.level_plan(m2, configs.level_spec(configs.config0()))
    assert a.pop("lattice") == 1 and b.pop("lattice") == 0  # arrays carry no refined-box metadata
    assert a == b


def test_optimal_samples_known_answers():
    """reference tests/test_mlmc.cpp:89-96"""
    assert wavemc.optimal_samples([1.0, 0.25], [1.0, 4.0], 1.0) == [4, 2]
    assert wavemc.optimal_samples([0.7], [5.0], 0.1) == [140]
    base = wavemc.optimal_samples([1.0, 0.3, 0.02], [1.0, 8.0, 64.0], 0.05)
    assert base == wavemc.optimal_samples([1.0, 0.3, 0.02], [100.0, 800.0, 6400.0], 0.05)
    with pytest.raises(wavemc.ConfigError):
        wavemc.optimal_samples([1.0], [0.0], 1.0)


def test_bias_proxy_known_answers():
    """reference tests/test_mlmc.cpp:137-142"""
    assert wavemc.bias_proxy_sq(0.0, 2.0) == 0.0
    assert wavemc.bias_proxy_sq(3e-5, 2.0) == pytest.approx(1e-10, rel=1e-12)
    assert wavemc.bias_proxy_sq(3e-5, 1.0) == pytest.approx(9.0 * wavemc.bias_proxy_sq(3e-5, 2.0), rel=1e-12)


def test_kl_modes_reproduce_the_cell_table():
    """wmc_kl_modes (the pointwise evaluator's mode list, used on the
    reference side for the per-element field) against wmc_kl_table."""
    import numpy as np
    from paper_2106_11117_b200 import configs, wavemc
    kl = configs.KL_FIELD
    table, _ = wavemc.kl_table(8, 8, kl["sigma"], kl["corr_len"], kl["modes"])
    modes = wavemc.kl_modes(kl["sigma"], kl["corr_len"], kl["modes"])

    def phi(omega, even, norm, t):
        return (np.cos(omega * t) if even else np.sin(omega * t)) / norm

    for iy in range(8):
        for ix in range(8):
            x, y = (ix + 0.5) / 8 - 0.5, (iy + 0.5) / 8 - 0.5
            row = [m[0] * phi(m[1], m[2], m[3], x) * phi(m[4], m[5], m[6], y) for m in modes]
            assert np.allclose(row, table[iy * 8 + ix], rtol=1e-13, atol=1e-15)


def test_tile_plan_streams_the_interior_of_a_mid_size_box():
    """Host-only plan of the temporally blocked step on a 257^2-node box at
    p = 8: thin side bands with corner squares and a streamed interior."""
    from paper_2106_11117_b200 import configs, wavemc
    d = configs.LevelDef(256, 8, 0.2 / 256, 8, configs.config1()[0].integrator)
    mesh = configs.build_mesh(d)
    spec = wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, final_time=8 * d.dt, batch=64)
    plan = wavemc.tile_plan(mesh, spec)
    assert plan["ok"] and plan["layout"] == "frame(24)+thin+stream"
    assert plan["n_tiles"] == 16 and plan["n_slabs"] == 1 and 0.6 < plan["streamed_frac"] < 0.75
    no_stream = wavemc.tile_plan(mesh, spec, stream=False)
    assert no_stream["ok"] and no_stream["n_slabs"] == 0 and no_stream["streamed_frac"] == 0.0


def test_per_element_field_level_plan():
    """One coefficient cell per triangle: no lattice form, same DOF counts."""
    from paper_2106_11117_b200 import configs, wavemc
    d = configs.config4()[0]
    mesh = configs.build_mesh(d)
    a = wavemc.level_plan(mesh, configs.level_spec(d, kl=True))
    b = wavemc.level_plan(mesh, configs.level_spec(d, kl="element"))
    assert a["lattice"] == 1 and b["lattice"] == 0
    assert (a["n"], a["n_r"], a["n_steps"]) == (b["n"], b["n_r"], b["n_steps"])
    assert b["nnz"] > a["nnz"]  # an entry per (pair, triangle)
