"""Config 2 on the device (graded L-shape, nested tiers): the HBM-resident
tier-stage kernels through the C ABI against the C restatement of the nested
scheme, and the reductions the reference pins (tests/test_config2_oracle.py).
Tolerances as the BASELINE north_star: per-sample QoI within 1e-10 relative,
per-level means and variances within 1e-9."""
import numpy as np
import pytest

from oracle_py import MeshArrays, problem
from paper_2106_11117_b200 import configs, wavemc

pytestmark = pytest.mark.gpu

QOI_RTOL = 1e-10
MOMENT_RTOL = 1e-9


def per_sample_rel(got, ref):
    got, ref = np.asarray(got), np.asarray(ref)
    return float(np.max(np.abs(got - ref) / np.abs(ref)))


def _oracle_problem(d, **kw):
    c = configs.CONFIG2_PROBLEM
    args = dict(final_time=d.final_time, cells=c["cells"], ic=c["ic"], box=c["qoi_box"], domain=c["domain"],
                qoi_mean=True, tiers=d.tiers)
    args.update(kw)
    dt = args.pop("dt", d.dt)
    p = args.pop("substeps", d.substeps)
    return problem(dt, p, 1, **args)


@pytest.fixture(scope="module")
def c2():
    defs = configs.config2(3)
    meshes = [configs.build_mesh(d) for d in defs]
    levels = [wavemc.Level(m, configs.level_spec(d)) for m, d in zip(meshes, defs)]
    arrays = [MeshArrays(*m.arrays()) for m in meshes]
    return defs, meshes, levels, arrays


def test_nested_path_selected(c2):
    _, _, levels, _ = c2
    for lv in levels:
        assert lv.info["substep_path"] == 4 and lv.info["tiers"] == 3
        r = lv.info["n_r_tier"]
        assert r[0] > r[1] > r[2] > 0


def test_config2_pairs_match_c_oracle(c2, coracle):
    defs, _, levels, arrays = c2
    for l, count in ((0, 8), (1, 4), (2, 2)):
        dq, qf, cost = wavemc.eval_pairs(levels[l], levels[l - 1] if l else None, 0, l, 0, count)
        pf = _oracle_problem(defs[l])
        pc = _oracle_problem(defs[l - 1]) if l else None
        rc, odq, oqf, _, _ = coracle.eval_pairs(arrays[l], pf, arrays[l - 1] if l else None, pc, 0, l, 0, count)
        assert rc == 0
        assert per_sample_rel(qf, oqf) < QOI_RTOL, l
        assert np.max(np.abs(dq - odq) / np.abs(oqf)) < 2 * QOI_RTOL, l
        if l == 0:
            p = defs[l].substeps
            assert cost["matvec_fine"] == count * (levels[l].info["n_steps"] - 1) * (p + p ** 2 + p ** 3)


def test_config2_single_tier_matches_reference(golden):
    """The device path on the config-2 mesh with one tier (P = P_1, p = 8):
    the reference's own LF-LTS on the same problem."""
    d = configs.config2()[0]
    g = golden("config2_reductions.json")["levels"][0]
    m = configs.build_mesh(d)
    for key in ("lts_single_tier", "lts_single_tier_nu0"):
        c = g[key]
        spec = configs.level_spec(d)
        spec.tiers, spec.substeps, spec.nu = 1, c["p"], c["nu"]
        lv = wavemc.Level(m, spec)
        assert lv.info["substep_path"] in (2, 3)
        _, qf, _ = wavemc.eval_pairs(lv, None, 0, c["stream_level"], c["first"], len(c["q"]))
        assert per_sample_rel(qf, c["q"]) < QOI_RTOL, key


def test_config2_leapfrog_matches_reference(golden):
    d = configs.config2()[0]
    c = golden("config2_reductions.json")["levels"][0]["lf"]
    spec = configs.level_spec(d)
    spec.tiers, spec.substeps, spec.integrator, spec.dt = 1, 1, wavemc.N.WMC_LEAPFROG, c["dt"]
    lv = wavemc.Level(configs.build_mesh(d), spec)
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 0, len(c["q"]))
    assert per_sample_rel(qf, c["q"]) < QOI_RTOL


def test_tiers_request_without_deeper_flags_is_single_tier():
    d = configs.config2()[0]
    xy, tri, fine, bnd = configs.build_mesh(d).arrays()
    m = wavemc.Mesh.from_arrays(xy, tri, np.minimum(fine, 1), bnd)
    spec = configs.level_spec(d)
    spec.dt = 0.05 / d.n_coarse
    one = wavemc.Level(m, spec)  # tiers requested, but P_2 = P_3 = {}: single tier
    assert one.info["tiers"] == 1
    spec1 = configs.level_spec(d)
    spec1.dt, spec1.tiers = spec.dt, 1
    ref = wavemc.Level(m, spec1)
    _, a, _ = wavemc.eval_pairs(one, None, 0, 0, 0, 64)
    _, b, _ = wavemc.eval_pairs(ref, None, 0, 0, 0, 64)
    assert np.array_equal(a, b)


def test_nested_all_rows_in_all_tiers_matches_c_oracle(coracle):
    """Every vertex in every tier: R_1 = R_2 = R_3 = all rows, no leap-frog
    rows in the sweep, every stage kernel covers the whole mesh."""
    d = configs.config2()[0]
    xy, tri, fine, bnd = configs.build_mesh(d).arrays()
    full = np.full_like(fine, 3)
    m = wavemc.Mesh.from_arrays(xy, tri, full, bnd)
    spec = configs.level_spec(d)
    spec.final_time = 0.25
    lv = wavemc.Level(m, spec)
    assert lv.info["n_r_tier"] == [lv.info["n"]] * 3
    _, qf, _ = wavemc.eval_pairs(lv, None, 0, 0, 5, 16)
    rc, _, oq, _, _ = coracle.eval_pairs(MeshArrays(xy, tri, full, bnd), _oracle_problem(d, final_time=0.25),
                                         None, None, 0, 0, 5, 16)
    assert rc == 0
    assert per_sample_rel(qf, oq) < QOI_RTOL


def test_config2_batches_and_repeats_bitwise(c2):
    _, meshes, levels, _ = c2
    d = configs.config2()[1]
    small = wavemc.Level(meshes[1], configs.level_spec(d, batch=64))
    _, a, _ = wavemc.eval_pairs(levels[1], levels[0], 9, 1, 0, 130)
    _, b, _ = wavemc.eval_pairs(small, levels[0], 9, 1, 0, 130)
    _, c, _ = wavemc.eval_pairs(levels[1], levels[0], 9, 1, 0, 130)
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_config2_fixed_mlmc_moments_match_c_oracle(c2, coracle):
    defs, _, levels, arrays = c2
    counts = [64, 16]
    stats = wavemc.run_mlmc_fixed(levels[:2], counts, seed=0)
    for l, n in enumerate(counts):
        pf = _oracle_problem(defs[l])
        pc = _oracle_problem(defs[l - 1]) if l else None
        rc, dq, qf, _, _ = coracle.eval_pairs(arrays[l], pf, arrays[l - 1] if l else None, pc, 0, l, 0, n)
        assert rc == 0
        ref = coracle.moments(dq, qf)
        for k in ("sum_dq", "sum_q", "variance", "mc_variance", "sum_dq2", "sum_q2"):
            assert stats[l][k] == pytest.approx(ref[k], rel=MOMENT_RTOL), (l, k)


def test_config2_instability_reported(coracle):
    """One tier with p = 2 cannot integrate the h/8 elements: the device
    reports the reference InstabilityError step like the oracle."""
    d = configs.config2()[0]
    m = configs.build_mesh(d)
    spec = configs.level_spec(d)
    spec.tiers = 1
    lv = wavemc.Level(m, spec)
    with pytest.raises(wavemc.NumericalError) as e:
        wavemc.eval_pairs(lv, None, 0, 0, 0, 4)
    rc, _, _, fi, fs = coracle.eval_pairs(MeshArrays(*m.arrays()), _oracle_problem(d, tiers=1), None, None, 0, 0,
                                          0, 4)
    assert rc == 3
    assert e.value.sample == fi and e.value.step == fs


def test_config2_wide_tier_stages_match_the_16_byte_form(c2):
    """Batches that are a multiple of 128 samples take tier_stage_wide_kernel
    (four samples per lane, 256-bit loads); the same samples in 64-sample
    batches take the 16-byte form.  Same per-sample products and sums."""
    defs, meshes, levels, _ = c2
    d = defs[2]
    small = wavemc.Level(meshes[2], configs.level_spec(d, batch=64))
    _, wide, _ = wavemc.eval_pairs(levels[2], None, 3, 2, 0, 256)
    _, narrow, _ = wavemc.eval_pairs(small, None, 3, 2, 0, 256)
    assert np.max(np.abs(wide - narrow) / np.abs(narrow)) < 1e-12
