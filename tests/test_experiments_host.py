"""The reference's own 1D sampling experiments (SURVEY.md section 8(f) row
2), host side: the restated hierarchy and the closed-form cost model against
the unmodified reference (tests/golden/experiments.json, generated through
its make_problem by oracle/make_golden.py --only-experiments)."""
import pytest

from paper_2106_11117_b200 import wavemc
from paper_2106_11117_b200._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING


@pytest.mark.parametrize("case", ["smooth1d_lts", "smooth1d_lf", "jump1d_lts", "jump1d_lf"])
def test_model_cost_matches_reference(golden, case):
    name, kind = case.split("_")
    integ = WMC_LOCAL_TIME_STEPPING if kind == "lts" else WMC_LEAPFROG
    assert wavemc.experiment_model_cost(name, integ) == golden("experiments.json")[case]["model_cost"]


def test_experiment_levels_plan(mesh1d):
    """Levels on the reference's own hierarchy meshes (wmc_mesh1d_create)."""
    prev = 0
    jm = mesh1d("jump1d")
    for level in range(5):
        info = wavemc.experiment_plan("jump1d", level, jm[level])
        assert info["nq"] == 512 and info["n"] > prev
        assert info["n"] == jm[level].n_vertices  # Neumann: every vertex a DOF
        prev = info["n"]
    # jump1d keeps a refined window to the last level (fine h = 1/512 < h0 / 16)
    assert info["p"] == 2 and info["n_r"] > 0
    # smooth1d is uniform on its last level (h0 / 16 = fine h)
    sm = mesh1d("smooth1d")
    assert wavemc.experiment_plan("smooth1d", 4, sm[4])["p"] == 1
    with pytest.raises(wavemc.ConfigError):
        wavemc.experiment_plan("smooth1d", 9, sm[4])
    with pytest.raises(wavemc.ConfigError):
        wavemc.Mesh1D([0.0, 1.0, 0.5], [0, 0], 0.5, 0.0)  # vertices not increasing


def test_channel_level_tables_from_reference_meshes():
    """Host side of the narrow-channel experiment on the reference's own
    meshes (tests/golden/channel): Neumann DOFs, LF-LTS ratio, per-sample
    cells and the line QoI, no device needed."""
    import os

    from paper_2106_11117_b200 import wavemc
    g = os.path.join(os.path.dirname(__file__), "golden", "channel")
    ov = dict(h0=0.05, fine_h=0.002, max_level=2, grid_n=64)
    for l, p in enumerate((25, 13, 7)):
        m = wavemc.Mesh.load(os.path.join(g, f"mesh_l{l}.txt.gz"))
        nv, nt, _, _ = m.info()
        info = wavemc.channel_plan(m, l, **ov)
        assert info["n"] == nv and info["p"] == p and info["nq"] == 64
        assert 0 < info["n_r"] < nv and info["n_recipes"] > 0
        lf = wavemc.channel_plan(m, l, integrator=0, **ov)
        assert lf["p"] == 1 and lf["n"] == nv
    cost = wavemc.experiment_model_cost("channel2d", **ov)
    assert cost == [34308.566617554192, 124605.34624289621, 628499.26331298659]  # the reference's make_problem
