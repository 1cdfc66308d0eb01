"""BASELINE.json configurations as mesh + level specifications.

The choices the BASELINE text leaves open are fixed here once and shared by
the GPU path and the oracles:
  * the refined square [0.45, 0.55]^2 is snapped outward to the level-0 grid
    (h = 1/16): [0.4375, 0.5625]^2 on every level;
  * c is U[0.5, 1.5) per cell of a 4x4 grid, drawn in row-major cell order
    k = iy*4 + ix from RngStream(seed=0, level, index) ("Philox" in the
    BASELINE text names the counter-based role; the reference generator is
    SplitMix64-keyed, rng.cpp:14-32);
  * fixed dt = 0.2 h_l for LF-LTS and 0.2 h_min for global leap-frog;
  * config 1 uses L = 4, i.e. five levels h_l = 1/16 .. 1/256 with
    p_l = 32, 16, 8, 4, 2, matching the five N_l values;
  * QoI: lumped quadrature of u(T) over the triangles whose centroid lies in
    [0.7, 0.9] x [0.4, 0.6].
Config 2 (graded L-shape, nested LTS; no reference counterpart):
  * h_l = 1/16 * 2^-l, l = 0..4 (L = 4 -> five levels, N_l = 32768 halving);
  * grading toward the re-entrant corner: leaf side s split while
    s > h sqrt(r / 0.25), three tiers h/2, h/4, h/8 (r < 1/4, 1/16, 1/64),
    each widened by one element layer; p = 2 per tier, dt = 0.2 h_l, T = 2;
  * c ~ U[0.5, 1.5) on an 8 x 8 grid over [-1, 1]^2 (row-major, the cells of
    the missing quadrant are drawn and unused);
  * u0 = exp(-((x + 0.5)^2 + (y - 0.5)^2) / 0.05^2) ("Gaussian pulse, width
    0.05", read as the initial condition as in SURVEY.md Appendix A item 8);
  * Q = mean of u(T) over the triangles with centroid in [0.4, 0.8]^2.
"""
from __future__ import annotations

from dataclasses import dataclass

from ._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING

FINE_LO, FINE_HI, SNAP = 0.45, 0.55, 1.0 / 16
H_MIN = 1.0 / 512

CONFIG1_COUNTS = [65536, 16384, 4096, 1024, 256]


@dataclass(frozen=True)
class LevelDef:
    n_coarse: int       # 1/h
    ratio: int          # h / h_min of this mesh (= p for LTS)
    dt: float
    substeps: int
    integrator: int
    final_time: float = 1.0
    shape: str = "square"  # "square" (configs 0, 1, 3, 4) or "lshape" (config 2)
    tiers: int = 1

    @property
    def h(self) -> float:
        return 1.0 / self.n_coarse


def config0() -> LevelDef:
    """Single-level MC: h = 1/32 refined by 4, p = 4, dt = 0.2 h, T = 1."""
    return LevelDef(32, 4, 0.2 / 32, 4, WMC_LOCAL_TIME_STEPPING)


def config0_leapfrog() -> LevelDef:
    return LevelDef(32, 4, 0.2 / 128, 1, WMC_LEAPFROG)


def config1(kind: str = "lts", n_levels: int = 5) -> list[LevelDef]:
    """MLMC, h_l = 1/16 * 2^-l, fixed h_min = 1/512, p_l = h_l / h_min."""
    out = []
    for l in range(n_levels):
        n_coarse = 16 << l
        ratio = 512 // n_coarse
        if kind == "lts":
            out.append(LevelDef(n_coarse, ratio, 0.2 / n_coarse, ratio, WMC_LOCAL_TIME_STEPPING))
        else:
            out.append(LevelDef(n_coarse, ratio, 0.2 * H_MIN, 1, WMC_LEAPFROG))
    return out


CONFIG2_COUNTS = [32768, 16384, 8192, 4096, 2048]
CONFIG2_TIERS = 3
CONFIG2_GRADE_RADIUS = 0.25
CONFIG2_PROBLEM = {"cells": (8, 8), "domain": (-1.0, 1.0, -1.0, 1.0), "ic": (-0.5, 0.5, 0.05 ** 2),
                   "qoi_box": (0.4, 0.8, 0.4, 0.8)}


def config2(n_levels: int = 5) -> list[LevelDef]:
    """Graded L-shape MLMC with nested LTS: 3 tiers, p = 2 per tier."""
    out = []
    for l in range(n_levels):
        n = 16 << l
        out.append(LevelDef(n, 1 << CONFIG2_TIERS, 0.2 / n, 2, WMC_LOCAL_TIME_STEPPING, final_time=2.0,
                            shape="lshape", tiers=CONFIG2_TIERS))
    return out


def config3() -> LevelDef:
    """Large batch: h = 1/1024, refined square at h/8, p = 8, T = 0.5."""
    return LevelDef(1024, 8, 0.2 / 1024, 8, WMC_LOCAL_TIME_STEPPING, final_time=0.5)


def config4() -> list[LevelDef]:
    """Adaptive MLMC, config-1 geometry, log-normal KL coefficient (see
    KL_FIELD); levels as config 1."""
    return config1()


# config 4 coefficient: c = exp(g), g = 0.5 * truncated KL (64 modes) of the
# separable exponential covariance exp(-|dx|/0.1 - |dy|/0.1), N(0,1) weights,
# sampled at the centres of a 32 x 32 cell grid (h = 1/32: a third of the
# correlation length; cell lines on mesh lines of every level)
KL_FIELD = {"cells": (32, 32), "sigma": 0.5, "corr_len": 0.1, "modes": 64}
CONFIG4_EPS = 1e-3

CONFIG0_COUNT = 1024
CONFIG3_COUNT = 8192


def build_mesh(d: LevelDef):
    from .wavemc import Mesh
    if d.shape == "lshape":
        return Mesh.build_lshape(d.n_coarse, d.tiers, CONFIG2_GRADE_RADIUS)
    return Mesh.build_square(d.n_coarse, d.ratio, FINE_LO, FINE_HI, SNAP)


def level_spec(d: LevelDef, device: int = 0, batch: int = 0, kl=False):
    """kl: False (uniform cells), True (config 4 on the KL cell grid) or
    "element" (config 4 with the field at every triangle's centroid)."""
    from .wavemc import LevelSpec
    if kl:
        from ._native import WMC_FIELD_LOGNORMAL_KL, WMC_FIELD_LOGNORMAL_KL_ELEMENT
        return LevelSpec(dt=d.dt, substeps=d.substeps, integrator=d.integrator, final_time=d.final_time,
                         device=device, batch=batch, cells_x=KL_FIELD["cells"][0], cells_y=KL_FIELD["cells"][1],
                         field=WMC_FIELD_LOGNORMAL_KL_ELEMENT if kl == "element" else WMC_FIELD_LOGNORMAL_KL,
                         kl_sigma=KL_FIELD["sigma"], kl_corr_len=KL_FIELD["corr_len"], kl_modes=KL_FIELD["modes"])
    if d.shape == "lshape":
        c = CONFIG2_PROBLEM
        return LevelSpec(dt=d.dt, substeps=d.substeps, integrator=d.integrator, final_time=d.final_time,
                         device=device, batch=batch, cells_x=c["cells"][0], cells_y=c["cells"][1], ic=c["ic"],
                         qoi_box=c["qoi_box"], domain=c["domain"], qoi_mean=True, tiers=d.tiers)
    return LevelSpec(dt=d.dt, substeps=d.substeps, integrator=d.integrator, final_time=d.final_time, device=device,
                     batch=batch)


def build_level(d: LevelDef, device: int = 0, batch: int = 0, kl=False):
    from .wavemc import Level
    return Level(build_mesh(d), level_spec(d, device, batch, kl))
