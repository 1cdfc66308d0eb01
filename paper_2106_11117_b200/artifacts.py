"""The reference's sampling-experiment artifacts from the device MLMC driver.

A user of the reference's `wavemc` CLI gets, per sampling experiment, the
files `run_sampling_experiment` writes (reference src/experiments.cpp:319-409):

  <exp>_<lf|lts>_eps<k>_levels.csv    per-level LevelStats (mlmc.hpp:75-84)
  <exp>_<lf|lts>_eps<k>_estimate.csv  the MLMC estimate on the output grid
  <exp>_work.csv                      one row per (integrator, eps)

each opened with the reference's header (`# wavemc 0.1.0` and the config echo
of src/config_io.cpp:227-256 minus `workers` / `out_dir`) and written at 17
significant digits.  This module writes the same files, same names, header,
columns and number format, from `wavemc.run_mlmc` on the device levels of the
1D experiments and of the narrow channel (reference meshes given).  Integer
columns (levels, sample counts, convergence, cost records) come out
identical to the reference's; floating-point columns agree to the parity
tolerance of the per-sample QoIs, not to the last digit (different summation
order on the device), so the files are format-compatible, not byte-identical.

Config files use the reference's flat `key = value` format with `#` comments
(src/config_io.cpp:109-224); `default_config` restates src/config_io.cpp:49-73.
"""
from __future__ import annotations

import dataclasses
import os
import sys
from dataclasses import dataclass, field

from . import wavemc
from ._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING

VERSION = "wavemc 0.1.0"  # the reference's kVersion (include/wavemc/experiments.hpp:20), first header line
EXPERIMENTS = ("smooth1d", "jump1d", "channel2d", "cost-sweep", "graded", "convergence")
SAMPLING = ("smooth1d", "jump1d", "channel2d")  # sampling experiments this framework evaluates on the device


@dataclass
class ExperimentConfig:
    """Reference ExperimentConfig (include/wavemc/experiments.hpp:24-54)."""
    experiment: str = "smooth1d"
    eps_list: list = field(default_factory=list)
    integrator: str = "both"  # lf | lts | both
    seed: int = 0
    workers: int = 1
    h0: float = 0.0
    fine_h: float = 0.0
    final_time: float = 0.0
    nu: float = 0.01
    safety: float = 0.9
    alpha: float = 2.0
    max_level: int = 4
    grid_n: int = 512
    initial_samples: int = 16
    bias_window: int = 1
    out_dir: str = "out"
    plot: bool = False
    sweep_axis: str = "r"
    sweep_lo: float = 0.0
    sweep_hi: float = 0.0
    sweep_count: int = 60
    dim: int = 1
    graded_s: float = 2.0
    graded_m_max: int = 4096


def default_config(experiment: str) -> ExperimentConfig:
    """Reference default_config (src/config_io.cpp:49-73)."""
    if experiment not in EXPERIMENTS:
        raise ValueError(f"unknown experiment {experiment!r}")
    c = ExperimentConfig(experiment=experiment)
    if experiment == "smooth1d":
        c.h0, c.fine_h, c.final_time, c.eps_list, c.max_level = 1 / 16, 1 / 256, 11.0, [4e-3, 2e-3, 1e-3], 4
    elif experiment == "jump1d":
        c.h0, c.fine_h, c.final_time, c.eps_list, c.max_level = 1 / 16, 1 / 512, 6.0, [4e-3, 2e-3, 1e-3], 4
    elif experiment == "channel2d":
        c.h0, c.fine_h, c.final_time, c.eps_list, c.max_level = 1 / 60, 7.6e-4, 1.0, [5e-5], 3
    elif experiment == "cost-sweep":
        c.dim, c.sweep_axis = 1, "r"
    elif experiment == "graded":
        c.dim, c.graded_s = 2, 2.0
    elif experiment == "convergence":
        c.final_time = 6.0
    return c


_KEYS = {f.name for f in dataclasses.fields(ExperimentConfig)} - {"eps_list"} | {"eps"}


def parse_config_text(text: str, experiment: str | None = None) -> ExperimentConfig:
    """Flat `key = value` config with `#` comments (reference
    parse_config_text, src/config_io.cpp:109-224): the experiment's defaults,
    then the file's values.  Unknown keys are an error naming them."""
    pairs = []
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"config: expected key = value, got {raw!r}")
        k, v = (s.strip() for s in line.split("=", 1))
        pairs.append((k, v))
    unknown = sorted({k for k, _ in pairs} - _KEYS)
    if unknown:
        raise ValueError("config: unknown keys: " + ", ".join(unknown))
    exp = experiment or dict(pairs).get("experiment", "smooth1d")
    c = default_config(exp)
    types = {f.name: f.type for f in dataclasses.fields(ExperimentConfig)}
    for k, v in pairs:
        if k == "experiment":
            if experiment is None:
                c.experiment = v
        elif k == "eps":
            c.eps_list = [float(x) for x in v.split(",") if x.strip()]
        elif types[k] in ("int", int):
            c.__dict__[k] = int(v)
        elif types[k] in ("float", float):
            c.__dict__[k] = float(v)
        elif types[k] in ("bool", bool):
            if v not in ("true", "false"):
                raise ValueError(f"config: {k} must be true or false")
            c.__dict__[k] = v == "true"
        else:
            c.__dict__[k] = v
    if c.integrator not in ("lf", "lts", "both"):
        raise ValueError("config: integrator must be lf, lts or both")
    return c


def _g(x: float) -> str:
    """A double as the reference's streams print it (setprecision(17), %.17g)."""
    return "%.17g" % x


def emit_config(c: ExperimentConfig) -> str:
    """Reference emit_config (src/config_io.cpp:227-256), same keys, order and format."""
    lines = [
        f"experiment = {c.experiment}",
        "eps = " + ",".join(_g(e) for e in c.eps_list),
        f"integrator = {c.integrator}",
        f"seed = {c.seed}",
        f"workers = {c.workers}",
        f"h0 = {_g(c.h0)}",
        f"fine_h = {_g(c.fine_h)}",
        f"final_time = {_g(c.final_time)}",
        f"nu = {_g(c.nu)}",
        f"safety = {_g(c.safety)}",
        f"alpha = {_g(c.alpha)}",
        f"max_level = {c.max_level}",
        f"grid_n = {c.grid_n}",
        f"initial_samples = {c.initial_samples}",
        f"bias_window = {c.bias_window}",
        f"out_dir = {c.out_dir}",
        "plot = " + ("true" if c.plot else "false"),
        f"sweep_axis = {c.sweep_axis}",
        f"sweep_lo = {_g(c.sweep_lo)}",
        f"sweep_hi = {_g(c.sweep_hi)}",
        f"sweep_count = {c.sweep_count}",
        f"dim = {c.dim}",
        f"graded_s = {_g(c.graded_s)}",
        f"graded_m_max = {c.graded_m_max}",
    ]
    return "\n".join(lines) + "\n"


def header(c: ExperimentConfig) -> str:
    """Reference write_header (src/experiments.cpp:319-332): the version and
    the config echo without the runtime knobs workers / out_dir."""
    out = [f"# {VERSION}"]
    for line in emit_config(c).splitlines():
        if line.startswith("workers") or line.startswith("out_dir"):
            continue
        out.append(f"# {line}")
    return "\n".join(out) + "\n"


def _open(c: ExperimentConfig, name: str):
    os.makedirs(c.out_dir, exist_ok=True)
    f = open(os.path.join(c.out_dir, name), "w", newline="\n")
    f.write(header(c))
    return f


def level_rows(result: wavemc.MlmcResult, alpha: float) -> list[dict]:
    """LevelStats as the reference's run_mlmc fills them (src/mlmc.cpp:208-226)."""
    rows = []
    for s in result.levels:
        l = s["level"]
        rows.append({"level": l, "n_samples": s["n_samples"], "variance": s["variance"],
                     "mc_variance": s["mc_variance"], "mean_dq_norm": abs(s["mean_dq"]),
                     "bias_proxy": wavemc.bias_proxy_sq(abs(s["mean_dq"]), alpha) if l >= 1 else 0.0,
                     "model_cost": s["model_cost"], **s["cost"]})
    return rows


def write_levels_csv(c: ExperimentConfig, name: str, result: wavemc.MlmcResult) -> None:
    """Reference write_levels_csv (src/experiments.cpp:344-355)."""
    with _open(c, name) as f:
        f.write("level,n_samples,variance,mc_variance,mean_dq_norm,bias_proxy,model_cost,"
                "matvec_full,matvec_fine,matvec_coarse,weighted_work\n")
        for r in level_rows(result, c.alpha):
            f.write(f"{r['level']},{r['n_samples']},{_g(r['variance'])},{_g(r['mc_variance'])},"
                    f"{_g(r['mean_dq_norm'])},{_g(r['bias_proxy'])},{_g(r['model_cost'])},"
                    f"{r['matvec_full']},{r['matvec_fine']},{r['matvec_coarse']},{r['weighted_work']}\n")


def grid_point(lo: float, hi: float, n: int, i: int) -> float:
    """Reference OutputGrid::point (include/wavemc/fem.hpp:22-23)."""
    return hi if i == n - 1 else lo + ((hi - lo) / (n - 1)) * i


def output_grid(experiment: str) -> tuple[float, float]:
    """The experiment's output grid (experiments.cpp: [0, kDomain1dLength] for
    the 1D experiments, [-kRectHalfHeight, kRectHalfHeight] for the channel)."""
    return (-0.5, 0.5) if experiment == "channel2d" else (0.0, 6.0)


def write_estimate_csv(c: ExperimentConfig, name: str, result: wavemc.MlmcResult) -> None:
    """Reference write_estimate_csv (src/experiments.cpp:357-363)."""
    est = result.estimate_vector
    lo, hi = output_grid(c.experiment)
    with _open(c, name) as f:
        f.write("point,value\n")
        for i in range(len(est)):
            f.write(f"{_g(grid_point(lo, hi, len(est), i))},{_g(float(est[i]))}\n")


def _overrides(c: ExperimentConfig, device: int) -> dict:
    return dict(h0=c.h0, fine_h=c.fine_h, final_time=c.final_time, nu=c.nu, safety=c.safety, grid_n=c.grid_n,
                max_level=c.max_level, device=device)


def run_sampling_experiment(c: ExperimentConfig, log=sys.stderr, device: int = 0, meshes=None) -> int:
    """Reference run_sampling_experiment (src/experiments.cpp:365-409) on the
    device: for each integrator (LF first, then LF-LTS) and each eps, the
    adaptive MLMC driver over the experiment's level hierarchy, then the
    levels / estimate CSVs and one row of <exp>_work.csv.  `meshes` holds the
    reference meshes of levels 0..max_level: wavemc.Mesh (channel2d, the
    reference's build_channel_mesh output) or wavemc.Mesh1D (smooth1d /
    jump1d, the reference's build_hierarchy levels with their ratios).
    Returns the reference's exit status (0 ok, 2 config error, 3 numerical
    failure)."""
    if c.experiment not in SAMPLING:
        log.write(f"config error: {c.experiment} is not a device sampling experiment here\n")
        return 2
    if meshes is None or len(meshes) < c.max_level + 1:
        log.write(f"config error: {c.experiment} needs the reference mesh of every level\n")
        return 2
    kinds = [k for k in ("lf", "lts") if c.integrator in (k, "both")]
    try:
        with _open(c, f"{c.experiment}_work.csv") as work:
            work.write("eps,integrator,converged,levels_used,total_model_cost,measured_work,"
                       "total_variance,bias_proxy\n")
            for kind in kinds:
                integ = WMC_LEAPFROG if kind == "lf" else WMC_LOCAL_TIME_STEPPING
                ov = _overrides(c, device)
                if c.experiment == "channel2d":
                    levels = [wavemc.Level.channel(meshes[l], l, integ, **ov) for l in range(c.max_level + 1)]
                else:
                    levels = [wavemc.Level.experiment(c.experiment, l, meshes[l], integ, **ov)
                              for l in range(c.max_level + 1)]
                costs = wavemc.experiment_model_cost(c.experiment, integ, **{k: v for k, v in ov.items()
                                                                                if k != "device"})
                for k, eps in enumerate(c.eps_list):
                    cfg = wavemc.MlmcConfig(eps=eps, alpha=c.alpha, initial_samples=c.initial_samples,
                                            max_level=c.max_level, master_seed=c.seed, bias_window=c.bias_window)
                    r = wavemc.run_mlmc(levels, costs, cfg)
                    log.write(f"{c.experiment} {kind} eps={_g(eps)} "
                              f"{'converged' if r.converged else 'NOT converged'}, levels 0..{r.levels_used}, "
                              f"model cost {r.total_model_cost:.6g}\n")
                    stem = f"{c.experiment}_{kind}_eps{k}"
                    write_levels_csv(c, stem + "_levels.csv", r)
                    write_estimate_csv(c, stem + "_estimate.csv", r)
                    measured = sum(s["cost"]["weighted_work"] for s in r.levels)
                    work.write(f"{_g(eps)},{kind},{1 if r.converged else 0},{r.levels_used},"
                               f"{_g(r.total_model_cost)},{measured},{_g(r.total_variance)},{_g(r.bias)}\n")
    except wavemc.ConfigError as e:  # noqa: F841
        log.write(f"config error: {e}\n")
        return 2
    except wavemc.NumericalError as e:
        log.write(f"numerical failure: {e}\n")
        return 3
    return 0
