"""The reference-side binding compiled and run (integration/reference_adapter.cpp,
built by oracle/Makefile `adapter` against the unmodified reference library
and the product library): the reference's OWN run_mlmc (src/mlmc.cpp:165-233)
drives the B200 evaluator through its MlmcProblem plug-in interface
(include/wavemc/mlmc.hpp:41-47) on BASELINE config 1 and must reproduce the
reference's own result (tests/golden/config1_adaptive.json: same N_l,
estimate and variances within 1e-9)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ADAPTER = os.path.join(ROOT, "oracle", "_ref", "reference_adapter")


@pytest.mark.skipif(not os.path.exists(ADAPTER), reason="reference adapter not built (oracle/Makefile adapter)")
def test_reference_run_mlmc_over_the_b200_evaluator(golden):
    g = golden("config1_adaptive.json")
    out = subprocess.run([ADAPTER, "--eps", repr(g["eps"]), "--block", "512"], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["device_calls"] > 0 and r["device_pairs"] >= sum(lv["N"] for lv in g["levels"])
    assert r["converged"] == g["converged"]
    assert [lv["N"] for lv in r["levels"]] == [lv["N"] for lv in g["levels"]]
    for got, want in zip(r["levels"], g["levels"]):
        assert got["variance"] == pytest.approx(want["variance"], rel=1e-9)
    assert r["estimate"] == pytest.approx(g["estimate"], rel=1e-9)
    assert r["total_variance"] == pytest.approx(g["total_variance"], rel=1e-9)
    assert r["bias"] == pytest.approx(g["bias"], rel=1e-9)
