"""Generate tests/golden/*.json from the UNMODIFIED reference library
(oracle/_ref/wavemc_ref_driver) -- run in the build container, where
/root/reference exists:  python oracle/make_golden.py [--only-round2 | --only-config1-full | --only-mesh1d | --only-config4 | --only-config2 | --only-cfl | --only-experiments | --only-artifacts | --only-channel]

The meshes come from the shared problem definition (the product's host mesh
builder), written in the reference fixture format (src/mesh_io.cpp:1-9) and
read back by the reference's load_trimesh, so geometry is never a parity
variable.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle_py import RefDriver, build  # noqa: E402

from paper_2106_11117_b200 import configs  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
CONFIG4_TIGHT_EPS = 1.5e-4


def dump(name, obj):
    os.makedirs(GOLDEN, exist_ok=True)
    with open(os.path.join(GOLDEN, name), "w") as f:
        json.dump(obj, f, indent=1)
        f.write("\n")


def config2_reductions(ref, tmp):
    """Config 2 (graded L-shape, nested tiers) has no reference counterpart;
    the reference pins its geometry, boundary, coefficient grid, IC and QoI
    through the two reductions it can run on the same mesh: single-tier LF-LTS
    with P = P_1 and p = 2^3 (stable at the finest tier), and global
    leap-frog at dt / 8."""
    c = configs.CONFIG2_PROBLEM
    args = {"cells-x": c["cells"][0], "cells-y": c["cells"][1], "ic": ",".join(map(repr, c["ic"])),
            "box": ",".join(map(repr, c["qoi_box"])), "domain": ",".join(map(repr, c["domain"])), "qoi-mean": 1,
            "T": 2.0}
    out = {"problem": {k: list(v) for k, v in c.items()}, "levels": []}
    meshes = {}
    for l, d in enumerate(configs.config2(3)):
        m = configs.build_mesh(d)
        path = os.path.join(tmp, f"config2_l{l}.mesh")
        m.dump(path)
        meshes[f"config2_l{l}"] = {"n_per_unit": d.n_coarse, "tiers": d.tiers, **ref.meshcheck(path)}
        if l > 0:
            continue
        p_fine = 2 ** d.tiers
        hdr, q = ref.solve(path, d.dt, p_fine, "lts", 0, 0, 8, **args)
        hdr_lf, q_lf = ref.solve(path, d.dt / p_fine, 1, "lf", 0, 0, 4, **args)
        hdr_nu0, q_nu0 = ref.solve(path, d.dt, p_fine, "lts", 1, 77, 4, nu=0.0, **args)
        out["levels"].append({
            "level": l, "n_per_unit": d.n_coarse, "dt": d.dt,
            "lts_single_tier": {"p": p_fine, "nu": 0.01, "stream_level": 0, "first": 0, "header": hdr,
                                "q": q.tolist()},
            "lts_single_tier_nu0": {"p": p_fine, "nu": 0.0, "stream_level": 1, "first": 77, "header": hdr_nu0,
                                    "q": q_nu0.tolist()},
            "lf": {"dt": d.dt / p_fine, "stream_level": 0, "first": 0, "header": hdr_lf, "q": q_lf.tolist()},
        })
    out["meshes"] = meshes
    dump("config2_reductions.json", out)


def cfl_samples(ref, tmp):
    """Per-sample CFL step: the reference's
    stable_dt recipe (src/experiments.cpp:30-43: power iteration at tol 1e-4
    from the level's c = 1 warm starts, margin 1.05, safety 0.9) replacing the
    fixed dt, on config 0 (LF-LTS and leap-frog) and config-1 pairs."""
    d0 = configs.config0()
    p0 = os.path.join(tmp, "cfl_config0.mesh")
    configs.build_mesh(d0).dump(p0)
    hdr, q = ref.solve(p0, d0.dt, d0.substeps, "lts", 0, 0, 8, cfl=0.9)
    hdr_lf, q_lf = ref.solve(p0, d0.dt, 1, "lf", 0, 0, 4, cfl=0.9)
    c1 = configs.config1()
    specs = []
    for l, d in enumerate(c1[:3]):
        p = os.path.join(tmp, f"cfl_config1_l{l}.mesh")
        configs.build_mesh(d).dump(p)
        specs.append((p, d.dt, d.substeps))
    pairs = ref.mlmc(specs, [4, 3, 2], per_sample=True, cfl=0.9)
    dump("cfl_samples.json", {"safety": 0.9, "config0_lts": {"q": q.tolist(), "header": hdr},
                              "config0_lf": {"q": q_lf.tolist(), "header": hdr_lf}, "config1_pairs": pairs})


def experiments(ref):
    """The reference's own 1D sampling experiments (SURVEY.md section 8(f)
    row 2) through its make_problem: per-sample QoI vectors of coupled pairs
    (every 4th of the 512 grid values plus the norms, to keep the fixture
    small) and run_mlmc at eps = 4e-3, for smooth1d / jump1d, LF-LTS / LF."""
    out = {}
    for name in ("smooth1d", "jump1d"):
        for kind in ("lts", "lf"):
            case = {"levels": []}
            for level, first in ((0, 0), (1, 5), (2, 11)):
                r = ref.experiment(name, kind, level=level, first=first, count=3)
                case["model_cost"] = r["model_cost"]
                samples = []
                for smp in r["samples"]:
                    dq, q = np.array(smp["dq"]), np.array(smp["q"])
                    w = np.full(len(q), 6.0 / (len(q) - 1))
                    w[0] = w[-1] = 0.5 * 6.0 / (len(q) - 1)
                    samples.append({"dq_every4": dq[::4].tolist(), "q_every4": q[::4].tolist(),
                                    "dq_norm": float(np.sqrt(np.sum(w * dq * dq))),
                                    "q_norm": float(np.sqrt(np.sum(w * q * q)))})
                case["levels"].append({"level": level, "first": first, "samples": samples})
            a = ref.experiment(name, kind, eps=4e-3)
            case["adaptive"] = {"eps": a["eps"], "converged": a["converged"], "total_variance": a["total_variance"],
                                "bias": a["bias"], "estimate_norm": a["estimate_norm"],
                                "estimate_every4": a["estimate"][::4], "levels": a["levels"],
                                "seconds": a["seconds"]}
            out[f"{name}_{kind}"] = case
    dump("experiments.json", out)


ARTIFACT_CONFIGS = {
    # small sampling runs of the reference's own experiments: two tolerances,
    # both integrators, a 64-point output grid, levels 0..3
    "smooth1d": "experiment = smooth1d\neps = 0.008,0.004\nintegrator = both\ngrid_n = 64\nmax_level = 3\n",
    "jump1d": "experiment = jump1d\neps = 0.008,0.004\nintegrator = both\ngrid_n = 64\nmax_level = 3\n",
    # the small channel hierarchy of tests/golden/channel (its meshes)
    "channel2d": ("experiment = channel2d\neps = 0.0004,0.0002\nintegrator = both\nh0 = 0.050000000000000003\n"
                  "fine_h = 0.002\ngrid_n = 64\nmax_level = 2\n"),
}


def artifacts(ref, tmp):
    """The reference's artifact files of its sampling experiments
    (run_experiment -> run_sampling_experiment, src/experiments.cpp:365-409):
    the config file and every CSV it writes, under tests/golden/artifacts/<exp>/."""
    import shutil
    for name, text in ARTIFACT_CONFIGS.items():
        dst = os.path.join(GOLDEN, "artifacts", name)
        shutil.rmtree(dst, ignore_errors=True)
        os.makedirs(dst)
        with open(os.path.join(dst, "experiment.cfg"), "w") as f:
            f.write(text)
        out = os.path.join(tmp, "art_" + name)
        cfg = os.path.join(tmp, name + ".cfg")
        with open(cfg, "w") as f:
            f.write(text + f"workers = {os.cpu_count() or 1}\nout_dir = {out}\n")
        ref.run("artifacts", "--config", cfg)
        for fn in sorted(os.listdir(out)):
            shutil.copy(os.path.join(out, fn), os.path.join(dst, fn))


CHANNEL = {"h0": 0.05, "fine_h": 0.002, "max_level": 2, "grid_n": 64}  # a small narrow-channel hierarchy


def channel(ref, tmp):
    """The reference's narrow-channel experiment (make_problem Channel2d,
    src/experiments.cpp:108-172) on a small hierarchy: the reference meshes of
    levels 0..2 (build_channel_mesh, gzip fixtures: the adapter's input),
    per-sample QoI vectors and cost records of coupled pairs for LF-LTS and
    LF, and run_mlmc at one tolerance."""
    import gzip
    import shutil
    c = CHANNEL
    dst = os.path.join(GOLDEN, "channel")
    os.makedirs(dst, exist_ok=True)
    for l in range(c["max_level"] + 1):
        path = os.path.join(tmp, f"channel_l{l}.mesh")
        ref.run("channel-mesh", "--h0", repr(c["h0"]), "--fine-h", repr(c["fine_h"]), "--level", l, "--out", path)
        with open(path, "rb") as f, open(os.path.join(dst, f"mesh_l{l}.txt.gz"), "wb") as raw, \
                gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as g:  # reproducible bytes
            shutil.copyfileobj(f, g)
    out = {"config": c}
    opts = {"h0": repr(c["h0"]), "fine-h": repr(c["fine_h"]), "max-level": c["max_level"], "grid-n": c["grid_n"]}
    for kind in ("lts", "lf"):
        case = {"levels": []}
        for level, first, count in ((0, 0, 6), (1, 3, 4), (2, 7, 3)):
            r = ref.experiment("channel2d", kind, level=level, first=first, count=count, **opts)
            case["model_cost"] = r["model_cost"]
            case["levels"].append({"level": level, "first": first, "samples": r["samples"]})
        a = ref.experiment("channel2d", kind, eps=2e-4, **opts)
        case["adaptive"] = {"eps": a["eps"], "converged": a["converged"], "total_variance": a["total_variance"],
                            "bias": a["bias"], "estimate_norm": a["estimate_norm"], "estimate": a["estimate"],
                            "levels": a["levels"], "seconds": a["seconds"]}
        out[kind] = case
    dump(os.path.join("channel", "channel.json"), out)


def hierarchies_1d(ref):
    """The reference's 1D mesh hierarchies of its smooth1d / jump1d
    experiments (build_state_1d -> build_hierarchy, src/experiments.cpp:62-85):
    the inputs the product takes through wmc_mesh1d_create, for the default
    configs (max_level 4; the artifact configs' max_level 3 is its prefix)."""
    dst = os.path.join(GOLDEN, "mesh1d")
    os.makedirs(dst, exist_ok=True)
    for name in ("smooth1d", "jump1d"):  # max_level 4; lower max_level: a prefix (nested bisection)
        h = json.loads(ref.run("hierarchy1d", "--name", name, "--max-level", 4))
        with open(os.path.join(dst, f"{name}_L4.json"), "w") as f:
            json.dump(h, f)
            f.write("\n")


def config1_full(ref, tmp):
    """Config-1 per-level sums, means and variances at the BASELINE N_l
    (65536 / 16384 / 4096 / 1024 / 256 coupled pairs) from the unmodified
    reference (sample_delta_q + LevelAccumulator + estimate_variance,
    src/mlmc.cpp:21-73, folded in (level, index) order as run_jobs does,
    :145-147).  About 75 core-minutes: run in the background."""
    c1 = configs.config1()
    specs = []
    for l, d in enumerate(c1):
        p = os.path.join(tmp, f"config1_l{l}.mesh")
        configs.build_mesh(d).dump(p)
        specs.append((p, d.dt, d.substeps))
    r = ref.mlmc(specs, configs.CONFIG1_COUNTS, timeout=6 * 3600)
    dump("config1_full_moments.json", r)


def round2(ref, tmp):
    """Round-2 fixtures: config 0 at its BASELINE 1024 samples (moments and
    per-sample Q); config-1 global leap-frog pairs at dt = 0.2 h_min on every
    level (BASELINE config 1's comparison arm; reference leapfrog_step,
    src/integrators.cpp:89-115); config 3's real mesh (h = 1/1024, square at
    h/8, p = 8) with T cut to 16 global steps."""
    d0 = configs.config0()
    p0 = os.path.join(tmp, "config0.mesh")
    configs.build_mesh(d0).dump(p0)
    mo = ref.mlmc([(p0, d0.dt, d0.substeps)], [configs.CONFIG0_COUNT], per_sample=True)
    dump("config0_moments_1024.json", mo)

    lf = configs.config1("lf")
    specs = []
    for l, d in enumerate(lf):
        p = os.path.join(tmp, f"config1_l{l}.mesh")
        configs.build_mesh(d).dump(p)
        specs.append((p, d.dt, d.substeps))
    pairs = ref.mlmc(specs, [4, 3, 3, 2, 2], kind="lf", per_sample=True)
    pairs["dt"] = lf[0].dt
    dump("config1_lf_pairs.json", pairs)

    d3 = configs.config3()
    p3 = os.path.join(tmp, "config3.mesh")
    configs.build_mesh(d3).dump(p3)
    t_cut = 16 * d3.dt
    hdr, q = ref.solve(p3, d3.dt, d3.substeps, "lts", 0, 0, 3, T=repr(t_cut))
    hdr2, q2 = ref.solve(p3, d3.dt, d3.substeps, "lts", 0, 4093, 2, T=repr(t_cut))
    # the BASELINE QoI box [0.7, 0.9] x [0.4, 0.6] is outside the domain of
    # dependence of the refined square within 16 steps, so the LTS substeps
    # are pinned through a second QoI over the refined square itself
    sq = "0.4375,0.5625,0.4375,0.5625"
    hdr3, q3 = ref.solve(p3, d3.dt, d3.substeps, "lts", 0, 0, 3, T=repr(t_cut), box=sq)
    t_long = 40 * d3.dt
    hdr4, q4 = ref.solve(p3, d3.dt, d3.substeps, "lts", 0, 7, 2, T=repr(t_long), box=sq)
    dump("config3_samples.json", {"dt": d3.dt, "p": d3.substeps, "nu": 0.01, "T": t_cut, "stream_level": 0,
                                  "header": hdr, "first": [0, 4093], "q": q.tolist() + q2.tolist(),
                                  "index": [0, 1, 2, 4093, 4094], "meshcheck": ref.meshcheck(p3),
                                  "square_box": {"box": [0.4375, 0.5625, 0.4375, 0.5625], "T": t_cut, "first": 0,
                                                 "header": hdr3, "q": q3.tolist()},
                                  "square_box_long": {"box": [0.4375, 0.5625, 0.4375, 0.5625], "T": t_long,
                                                      "first": 7, "header": hdr4, "q": q4.tolist()}})


def main():
    build()
    ref = RefDriver()
    tmp = tempfile.mkdtemp(prefix="wmc_golden_")
    if "--only-config2" in sys.argv:
        config2_reductions(ref, tmp)
        return
    if "--only-cfl" in sys.argv:
        cfl_samples(ref, tmp)
        return
    if "--only-experiments" in sys.argv:
        experiments(ref)
        return
    if "--only-artifacts" in sys.argv:
        artifacts(ref, tmp)
        return
    if "--only-config1-full" in sys.argv:
        config1_full(ref, tmp)
        return
    if "--only-config4" in sys.argv:
        config4(ref, tmp)
        return
    if "--only-mesh1d" in sys.argv:
        hierarchies_1d(ref)
        return
    if "--only-round2" in sys.argv:
        round2(ref, tmp)
        return
    if "--only-channel" in sys.argv:
        channel(ref, tmp)
        return

    # RNG words and uniform draws (rng.hpp:14-19, rng.cpp:14-32)
    streams = [(0, 0, 0), (0, 1, 7), (12345, 3, 987654321), (2**63 + 5, 4, 2**40 + 3)]
    dump("rng.json", {
        "words": [{"seed": s, "level": l, "index": i, "words": [hex(w) for w in ref.rng(s, l, i, 6)]}
                  for s, l, i in streams],
        "uniform": [{"seed": s, "level": l, "index": i, "lo": 0.5, "hi": 1.5,
                     "values": ref.rng(s, l, i, 16, uniform=True)} for s, l, i in streams],
    })

    # Chebyshev constants (integrators.cpp:34-66)
    cases = [(1, 0.0), (2, 0.0), (2, 0.01), (4, 0.01), (8, 0.01), (16, 0.01), (32, 0.01), (32, 0.0), (5, 0.5)]
    dump("chebyshev.json", [{"p": p, "nu": nu, **dict(zip(["delta", "omega", "beta_int", "beta_half"],
                                                            ref.consts(p, nu)))} for p, nu in cases])

    # meshes: reference check_mesh report (mesh2d.cpp:415-452)
    defs = {"config0": configs.config0()}
    for l, d in enumerate(configs.config1()):
        defs[f"config1_l{l}"] = d
    paths = {}
    meshes = {}
    for name, d in defs.items():
        m = configs.build_mesh(d)
        p = os.path.join(tmp, name + ".mesh")
        m.dump(p)
        paths[name] = p
        meshes[name] = {"n_coarse": d.n_coarse, "ratio": d.ratio, **ref.meshcheck(p)}
    dump("meshes.json", meshes)

    # config 0 level data: z0, lumped mass, QoI weights (interior vertex order)
    d0 = configs.config0()
    vid, z0, mass, w = ref.level(paths["config0"], d0.dt, d0.substeps)
    dump("config0_level.json", {"interior_vertex": vid.tolist(), "z0": z0.tolist(), "mass": mass.tolist(),
                                "qoi_w": w.tolist()})

    # config 0 per-sample QoI, LF-LTS and global leap-frog
    hdr, q = ref.solve(paths["config0"], d0.dt, d0.substeps, "lts", 0, 0, 32)
    lf = configs.config0_leapfrog()
    hdr_lf, q_lf = ref.solve(paths["config0"], lf.dt, 1, "lf", 0, 0, 8)
    # nu = 0 and a non-zero first index / stream level
    hdr_nu0, q_nu0 = ref.solve(paths["config0"], d0.dt, d0.substeps, "lts", 2, 1000, 8, nu=0.0)
    dump("config0_samples.json", {
        "lts": {"dt": d0.dt, "p": d0.substeps, "nu": 0.01, "stream_level": 0, "first": 0, "header": hdr,
                "q": q.tolist()},
        "lf": {"dt": lf.dt, "p": 1, "stream_level": 0, "first": 0, "header": hdr_lf, "q": q_lf.tolist()},
        "lts_nu0": {"dt": d0.dt, "p": d0.substeps, "nu": 0.0, "stream_level": 2, "first": 1000, "header": hdr_nu0,
                    "q": q_nu0.tolist()},
    })

    # config 0 MLMC moments over 256 samples (single level)
    mo = ref.mlmc([(paths["config0"], d0.dt, d0.substeps)], [256], per_sample=True)
    dump("config0_moments.json", mo)

    # config 1 coupled pairs on every level, per-sample dQ and Q_fine
    c1 = configs.config1()
    specs = [(paths[f"config1_l{l}"], d.dt, d.substeps) for l, d in enumerate(c1)]
    pairs = ref.mlmc(specs, [6, 6, 4, 3, 2], per_sample=True)
    dump("config1_pairs.json", pairs)

    # adaptive Giles driver (reference run_mlmc) on the config-1 hierarchy;
    # model cost = DOF-updates of one solve on the level
    adaptive = ref.adaptive(specs, 2e-4)
    adaptive["eps"] = 2e-4
    adaptive["model_cost"] = [lv["n"] + (lv["n_steps"] - 1) * (lv["n"] + (d.substeps - 1) * lv["n_r"])
                              for lv, d in zip(pairs["levels"], c1)]
    dump("config1_adaptive.json", adaptive)

    config4(ref, tmp, specs, adaptive["model_cost"])
    config2_reductions(ref, tmp)
    cfl_samples(ref, tmp)
    experiments(ref)
    print("golden fixtures written to", GOLDEN)


def config4(ref, tmp, specs=None, model_cost=None):
    """Config 4: log-normal KL coefficient on the KL_FIELD cell grid (new
    field, our shared definition), solved by the reference: coupled pairs and
    the reference run_mlmc at the BASELINE RMSE target."""
    from paper_2106_11117_b200 import wavemc
    if specs is None:
        c1 = configs.config1()
        specs = []
        for l, d in enumerate(c1):
            p = os.path.join(tmp, f"config1_l{l}.mesh")
            configs.build_mesh(d).dump(p)
            specs.append((p, d.dt, d.substeps))
        model_cost = json.load(open(os.path.join(GOLDEN, "config1_adaptive.json")))["model_cost"]
    kl = configs.KL_FIELD
    table, lam = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
    tpath = os.path.join(tmp, "kl.txt")
    with open(tpath, "w") as f:
        f.write(f"{table.shape[0]} {table.shape[1]}\n")
        f.write("\n".join(repr(float(v)) for v in table.ravel()))
        f.write("\n")
    klargs = {"kl-table": tpath, "cells-x": kl["cells"][0], "cells-y": kl["cells"][1]}
    kl_pairs = ref.mlmc(specs[:3], [4, 3, 2], per_sample=True, **klargs)
    kl_pairs["kl_lambda_sum"] = float(lam.sum())
    dump("config4_pairs.json", kl_pairs)
    kl_adaptive = ref.adaptive(specs, configs.CONFIG4_EPS, **klargs)
    kl_adaptive["eps"] = configs.CONFIG4_EPS
    kl_adaptive["model_cost"] = model_cost
    kl_adaptive["cells"] = list(kl["cells"])
    # a tighter target, so the driver adds samples and levels beyond the warm-up
    tight = ref.adaptive(specs, CONFIG4_TIGHT_EPS, **klargs)
    tight["eps"] = CONFIG4_TIGHT_EPS
    kl_adaptive["tight"] = tight
    dump("config4_adaptive.json", kl_adaptive)
    # the field at every triangle's centroid: the reference's assemble calls
    # speed2(x, y) = exp(g(x, y)) itself (fem.cpp:103-104), g from the shared mode list
    modes = wavemc.kl_modes(kl["sigma"], kl["corr_len"], kl["modes"])
    mpath = os.path.join(tmp, "kl_modes.txt")
    with open(mpath, "w") as f:
        f.write(f"{modes.shape[0]}\n")
        f.write("\n".join(repr(float(v)) for v in modes.ravel()))
        f.write("\n")
    elargs = {"kl-modes": mpath}
    el = {"pairs": ref.mlmc(specs[:3], [4, 3, 2], per_sample=True, **elargs)}
    el["adaptive"] = ref.adaptive(specs, configs.CONFIG4_EPS, **elargs)
    el["adaptive"]["eps"] = configs.CONFIG4_EPS
    el["tight"] = ref.adaptive(specs, CONFIG4_TIGHT_EPS, **elargs)
    el["tight"]["eps"] = CONFIG4_TIGHT_EPS
    el["model_cost"] = model_cost
    # one coupled pair on each of the five levels (levels 3-4: more than 32 k
    # triangles, the per-entry cell arrays of the sweep and the substeps)
    el["pairs_all_levels"] = ref.mlmc(specs, [1, 1, 1, 1, 1], per_sample=True, **elargs)
    dump("config4_element.json", el)


if __name__ == "__main__":
    main()
