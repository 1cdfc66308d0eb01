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


def test_experiment_levels_plan():
    prev = 0
    for level in range(5):
        info = wavemc.experiment_plan("jump1d", level)
        assert info["nq"] == 512 and info["n"] > prev
        prev = info["n"]
    # jump1d keeps a refined window to the last level (fine h = 1/512 < h0 / 16)
    assert info["p"] == 2 and info["n_r"] > 0
    # smooth1d is uniform on its last level (h0 / 16 = fine h)
    assert wavemc.experiment_plan("smooth1d", 4)["p"] == 1
    with pytest.raises(wavemc.ConfigError):
        wavemc.experiment_plan("smooth1d", 9)
