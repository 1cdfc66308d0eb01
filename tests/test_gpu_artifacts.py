"""The reference's sampling-experiment artifacts written from the device
MLMC driver (paper_2106_11117_b200.artifacts) against the files the
unmodified reference wrote for the same config (tests/golden/artifacts):
same file set, headers and columns; integer columns identical (same N_l,
levels, convergence, matvec counts); floating-point columns within the
per-level estimator tolerance (1e-9 relative)."""
import csv
import io
import os

import pytest

from paper_2106_11117_b200 import artifacts

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "artifacts")
RTOL = 1e-9


def _read(path):
    with open(path) as f:
        text = f.read()
    head = "".join(line + "\n" for line in text.splitlines() if line.startswith("#"))
    body = "\n".join(line for line in text.splitlines() if not line.startswith("#"))
    rows = list(csv.DictReader(io.StringIO(body)))
    return head, rows


def _close(a, b, scale=None):
    a, b = float(a), float(b)
    return abs(a - b) <= RTOL * (scale if scale is not None else max(abs(a), abs(b), 1e-300))


@pytest.mark.parametrize("name", sorted(os.listdir(GOLDEN)))
def test_artifacts_match_reference(name, tmp_path, mesh1d):
    with open(os.path.join(GOLDEN, name, "experiment.cfg")) as f:
        c = artifacts.parse_config_text(f.read())
    c.out_dir = str(tmp_path)
    log = io.StringIO()
    from paper_2106_11117_b200 import wavemc
    if c.experiment == "channel2d":  # the reference meshes of the small channel hierarchy
        meshes = [wavemc.Mesh.load(os.path.join(GOLDEN, "..", "channel", f"mesh_l{l}.txt.gz"))
                  for l in range(c.max_level + 1)]
    else:  # the reference's 1D hierarchy
        meshes = mesh1d(c.experiment, c.max_level)
    assert artifacts.run_sampling_experiment(c, log, meshes=meshes) == 0, log.getvalue()
    want_files = sorted(fn for fn in os.listdir(os.path.join(GOLDEN, name)) if fn.endswith(".csv"))
    assert sorted(os.listdir(tmp_path)) == want_files
    for fn in want_files:
        gh, got = _read(os.path.join(tmp_path, fn))
        wh, want = _read(os.path.join(GOLDEN, name, fn))
        assert gh == wh, fn
        assert len(got) == len(want) and got[0].keys() == want[0].keys(), fn
        if fn.endswith("_levels.csv"):
            for g, w in zip(got, want):
                for k in ("level", "n_samples", "matvec_full", "matvec_fine", "matvec_coarse", "weighted_work"):
                    assert g[k] == w[k], (fn, k, g[k], w[k])
                for k in ("variance", "mc_variance", "mean_dq_norm", "bias_proxy", "model_cost"):
                    assert _close(g[k], w[k]), (fn, k, g[k], w[k])
        elif fn.endswith("_estimate.csv"):
            scale = max(abs(float(w["value"])) for w in want)
            for g, w in zip(got, want):
                assert g["point"] == w["point"]
                assert _close(g["value"], w["value"], scale), (fn, g, w)
        else:
            for g, w in zip(got, want):
                for k in ("eps", "integrator", "converged", "levels_used", "measured_work"):
                    assert g[k] == w[k], (fn, k, g[k], w[k])
                for k in ("total_model_cost", "total_variance", "bias_proxy"):
                    assert _close(g[k], w[k]), (fn, k, g[k], w[k])
