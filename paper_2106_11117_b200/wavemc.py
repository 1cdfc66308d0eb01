"""Host-side mirror of the reference sampler API over the B200 C ABI.

Reference interface this mirrors (paths in /root/reference/proj):
  * MlmcProblem / sample_delta_q / run_jobs  include/wavemc/mlmc.hpp:41-51,
    src/mlmc.cpp:21-37, :107-149  ->  Level + eval_pairs (batched pairs)
  * LevelAccumulator / estimate_variance     include/wavemc/mlmc.hpp:53-73
    ->  LevelStats fields (sum_dq, sum_dq2, sum_q, sum_q2, variance, ...)
  * run_mlmc / MlmcConfig / MlmcResult       include/wavemc/mlmc.hpp:14-112
    ->  run_mlmc, run_mlmc_fixed
  * RngStream(seed, level, index)            include/wavemc/rng.hpp:27-46
    ->  draw_cells (device draws, bit-identical)
  * errors: ConfigError (exit 2), NumericalError / InstabilityError{step}
    (exit 3)                                 include/wavemc/errors.hpp:9-26
All compute runs in libwavemc_b200.so on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import ConfigError, DeviceError, NumericalError, WavemcError  # noqa: F401


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Mesh:
    """A triangulation of the unit square (TriMesh, reference mesh.hpp:48-74)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    @classmethod
    def build_square(cls, n_coarse: int, ratio: int, fine_lo: float = 0.45, fine_hi: float = 0.55,
                     snap: float = 1.0 / 16, small_factor: float = 0.7) -> "Mesh":
        spec = N.SquareMeshSpec(n_coarse, ratio, fine_lo, fine_hi, snap, small_factor)
        h = C.c_void_p()
        N.check(N.lib().wmc_mesh_build_square(C.byref(spec), C.byref(h)))
        return cls(h.value)

    @classmethod
    def build_lshape(cls, n_per_unit: int, tiers: int = 3, grade_radius: float = 0.25) -> "Mesh":
        """Graded L-shape [-1,1]^2 minus [0,1]x[-1,0] (BASELINE config 2); flags = tiers."""
        spec = N.LShapeMeshSpec(n_per_unit, tiers, grade_radius)
        h = C.c_void_p()
        N.check(N.lib().wmc_mesh_build_lshape(C.byref(spec), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, xy, tri, fine, boundary, coarse_h=0.0, fine_h=0.0) -> "Mesh":
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        fine = np.ascontiguousarray(fine, dtype=np.uint8)
        boundary = np.ascontiguousarray(boundary, dtype=np.uint8)
        h = C.c_void_p()
        N.check(N.lib().wmc_mesh_create(len(xy), len(tri), _dptr(xy), tri.ctypes.data_as(C.POINTER(C.c_int)),
                                        fine.ctypes.data_as(C.POINTER(C.c_ubyte)),
                                        boundary.ctypes.data_as(C.POINTER(C.c_ubyte)), coarse_h, fine_h,
                                        C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, path: str) -> "Mesh":
        """A mesh in the reference's plain-text fixture format (src/mesh_io.cpp:
        1-9, 47-90: `wavemc-mesh-2d nv nt coarse_h fine_h`, `v x y`, `t a b c flag`),
        e.g. the reference's build_channel_mesh output; gzip-compressed files
        (*.gz) too.  No vertex is marked Dirichlet (Neumann problems)."""
        import gzip
        opener = gzip.open if str(path).endswith(".gz") else open
        with opener(path, "rt") as f:
            head = f.readline().split()
            if len(head) != 5 or head[0] != "wavemc-mesh-2d":
                raise ValueError(f"{path}: not a wavemc-mesh-2d fixture")
            nv, nt = int(head[1]), int(head[2])
            coarse_h, fine_h = float(head[3]), float(head[4])
            xy = np.zeros((nv, 2), np.float64)
            tri = np.zeros((nt, 3), np.int32)
            fine = np.zeros(nt, np.uint8)
            for i in range(nv):
                tag, x, y = f.readline().split()
                xy[i] = float(x), float(y)
            for t in range(nt):
                tag, a, b, c, flag = f.readline().split()
                tri[t] = int(a), int(b), int(c)
                fine[t] = int(flag)
        return cls.from_arrays(xy, tri, fine, np.zeros(nv, np.uint8), coarse_h, fine_h)

    def info(self):
        nv, nt = C.c_int(), C.c_int()
        ch, fh = C.c_double(), C.c_double()
        N.check(N.lib().wmc_mesh_info(self._h, C.byref(nv), C.byref(nt), C.byref(ch), C.byref(fh)))
        return nv.value, nt.value, ch.value, fh.value

    def arrays(self):
        nv, nt, _, _ = self.info()
        xy = np.zeros((nv, 2), np.float64)
        tri = np.zeros((nt, 3), np.int32)
        fine = np.zeros(nt, np.uint8)
        boundary = np.zeros(nv, np.uint8)
        N.check(N.lib().wmc_mesh_export(self._h, _dptr(xy), tri.ctypes.data_as(C.POINTER(C.c_int)),
                                        fine.ctypes.data_as(C.POINTER(C.c_ubyte)),
                                        boundary.ctypes.data_as(C.POINTER(C.c_ubyte))))
        return xy, tri, fine, boundary

    def dump(self, path: str) -> None:
        N.check(N.lib().wmc_mesh_dump(self._h, str(path).encode()))

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            N.lib().wmc_mesh_destroy(self._h)
            self._h = C.c_void_p()


@dataclass
class LevelSpec:
    """Per-level problem definition (wmc_level_desc)."""
    dt: float
    substeps: int = 1
    integrator: int = N.WMC_LOCAL_TIME_STEPPING
    final_time: float = 1.0
    nu: float = 0.01
    cells_x: int = 4
    cells_y: int = 4
    coef_lo: float = 0.5
    coef_hi: float = 1.5
    ic: tuple = (0.3, 0.5, 0.01)
    qoi_box: tuple = (0.7, 0.9, 0.4, 0.6)
    device: int = 0
    batch: int = 0
    field: int = N.WMC_FIELD_UNIFORM
    kl_sigma: float = 0.5
    kl_corr_len: float = 0.1
    kl_modes: int = 64
    tiers: int = 1
    domain: tuple = (0.0, 1.0, 0.0, 1.0)
    qoi_mean: bool = False
    cfl_safety: float = 0.0  # > 0: per-sample dt (reference stable_dt recipe)

    def desc(self) -> N.LevelDesc:
        d = N.LevelDesc()
        N.lib().wmc_level_desc_default(C.byref(d))
        d.cells_x, d.cells_y = self.cells_x, self.cells_y
        d.coef_lo, d.coef_hi = self.coef_lo, self.coef_hi
        d.final_time, d.dt, d.substeps, d.nu = self.final_time, self.dt, self.substeps, self.nu
        d.integrator = self.integrator
        d.ic_x, d.ic_y, d.ic_width2 = self.ic
        for i, v in enumerate(self.qoi_box):
            d.qoi_box[i] = v
        d.device, d.batch = self.device, self.batch
        d.field, d.kl_sigma, d.kl_corr_len, d.kl_modes = self.field, self.kl_sigma, self.kl_corr_len, self.kl_modes
        d.tiers = self.tiers
        for i, v in enumerate(self.domain):
            d.domain[i] = v
        d.qoi_mean = 1 if self.qoi_mean else 0
        d.cfl_safety = self.cfl_safety
        return d


def _info_dict(info: N.LevelInfo) -> dict:
    out = {k: getattr(info, k) for k, _ in N.LevelInfo._fields_}
    out["n_r_tier"] = list(out["n_r_tier"])[: max(out["tiers"], 1)]
    return out


def experiment_desc(experiment: str, integrator: int = N.WMC_LOCAL_TIME_STEPPING, **overrides) -> N.ExperimentDesc:
    """The reference's default_config for a 1D experiment (src/config_io.cpp:49-73) with overrides."""
    kind = {"smooth1d": N.WMC_EXP_SMOOTH1D, "jump1d": N.WMC_EXP_JUMP1D, "channel2d": N.WMC_EXP_CHANNEL2D}[experiment]
    d = N.ExperimentDesc()
    N.lib().wmc_experiment_desc_default(C.byref(d), kind)
    d.integrator = integrator
    for k, v in overrides.items():
        setattr(d, k, v)
    return d


class Mesh1D:
    """A 1D mesh of the reference's sampling experiments (wmc_mesh1d): the
    reference's Mesh1D (include/wavemc/mesh.hpp:21-33) as arrays, one level of
    its build_hierarchy (src/mesh1d.cpp:76-125) with that level's ratio p_l."""

    def __init__(self, vertices, fine_flags, coarse_h: float, fine_h: float, ratio: int = 1):
        v = np.ascontiguousarray(vertices, np.float64)
        f = np.ascontiguousarray(fine_flags, np.uint8)
        if f.shape != (len(v) - 1,):
            raise ValueError("Mesh1D: one fine flag per element")
        h = C.c_void_p()
        N.check(N.lib().wmc_mesh1d_create(len(v), _dptr(v), f.ctypes.data_as(C.POINTER(C.c_ubyte)), coarse_h, fine_h,
                                          C.byref(h)))
        self._h = h
        self.ratio = int(ratio)
        self.n_vertices = len(v)

    @classmethod
    def hierarchy(cls, levels: list[dict]) -> list["Mesh1D"]:
        """Meshes from the reference hierarchy's levels, each a dict with
        vertices, fine_flags, coarse_h, fine_h and ratio (the reference's
        MeshHierarchy: levels[l] and ratios[l])."""
        return [cls(lv["vertices"], lv["fine_flags"], lv["coarse_h"], lv["fine_h"], lv["ratio"]) for lv in levels]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().wmc_mesh1d_destroy(h)
            self._h = None


def experiment_plan(experiment: str, level: int, mesh: Mesh1D, integrator: int = N.WMC_LOCAL_TIME_STEPPING,
                    **overrides) -> dict:
    """Host-only sizes of one experiment level on `mesh` (that level's mesh)."""
    info = N.LevelInfo()
    N.check(N.lib().wmc_experiment_plan(mesh._h, mesh.ratio, C.byref(experiment_desc(experiment, integrator, **overrides)),
                                        level, C.byref(info)))
    return _info_dict(info)


def experiment_model_cost(experiment: str, integrator: int = N.WMC_LOCAL_TIME_STEPPING, **overrides) -> list[float]:
    """The reference's closed-form model cost of every level (run_mlmc weights)."""
    d = experiment_desc(experiment, integrator, **overrides)
    return [N.lib().wmc_experiment_model_cost(C.byref(d), l) for l in range(d.max_level + 1)]


def channel_plan(mesh: Mesh, level: int, integrator: int = N.WMC_LOCAL_TIME_STEPPING, **overrides) -> dict:
    """Host-only sizes of one channel level on `mesh` (no device)."""
    info = N.LevelInfo()
    N.check(N.lib().wmc_channel_plan(mesh._h, C.byref(experiment_desc("channel2d", integrator, **overrides)), level,
                                     C.byref(info)))
    return _info_dict(info)


def level_plan(mesh: Mesh, spec: LevelSpec) -> dict:
    """Host-only level tables: sizes and DOF-update counts (no device)."""
    d = spec.desc()
    info = N.LevelInfo()
    N.check(N.lib().wmc_level_plan(mesh._h, C.byref(d), C.byref(info)))
    return _info_dict(info)


def tile_plan(mesh: Mesh, spec: LevelSpec, stream: bool = True) -> dict:
    """Host-only plan of the temporally blocked step (wmc_tile_plan): tiles
    around the box ring, streamed slabs inside; no device."""
    d = spec.desc()
    info = N.TilePlanInfo()
    N.check(N.lib().wmc_tile_plan(mesh._h, C.byref(d), 1 if stream else 0, C.byref(info)))
    return {"ok": bool(info.ok), "n_tiles": info.n_tiles, "n_slabs": info.n_slabs, "max_gen": info.max_gen,
            "work_factor": info.work_factor, "streamed_frac": info.streamed_frac,
            "layout": info.layout.decode(), "reason": info.reason.decode()}


class Level:
    """One MLMC level resident on a device (wmc_level)."""

    def __init__(self, mesh: Mesh, spec: LevelSpec):
        self.mesh = mesh
        self.spec = spec
        d = spec.desc()
        h = C.c_void_p()
        N.check(N.lib().wmc_level_create(mesh._h, C.byref(d), C.byref(h)))
        self._h = h
        info = N.LevelInfo()
        N.check(N.lib().wmc_level_get_info(self._h, C.byref(info)))
        self.info = _info_dict(info)

    @classmethod
    def experiment(cls, experiment: str, level: int, mesh: Mesh1D, integrator: int = N.WMC_LOCAL_TIME_STEPPING,
                   **overrides):
        """Level `level` of the reference's own 1D sampling experiment
        ("smooth1d" or "jump1d"; reference make_problem, src/experiments.cpp:56-106)
        on `mesh`, the reference hierarchy's mesh of that level (with its ratio),
        reference default_config unless overridden (h0, fine_h, final_time, nu,
        safety, grid_n, max_level, device, batch)."""
        d = experiment_desc(experiment, integrator, **overrides)
        self = cls.__new__(cls)
        self.mesh = mesh
        self.spec = None
        self.experiment_desc = d
        h = C.c_void_p()
        N.check(N.lib().wmc_level_create_experiment(mesh._h, mesh.ratio, C.byref(d), level, C.byref(h)))
        self._h = h
        info = N.LevelInfo()
        N.check(N.lib().wmc_level_get_info(self._h, C.byref(info)))
        self.info = _info_dict(info)
        return self

    @classmethod
    def channel(cls, mesh: "Mesh", level: int, integrator: int = N.WMC_LOCAL_TIME_STEPPING, **overrides):
        """Level `level` of the reference's narrow-channel experiment on `mesh`,
        the reference's build_channel_mesh of that level (make_problem
        Channel2d, src/experiments.cpp:108-172; wmc_level_create_channel)."""
        d = experiment_desc("channel2d", integrator, **overrides)
        self = cls.__new__(cls)
        self.mesh = mesh
        self.spec = None
        self.experiment_desc = d
        h = C.c_void_p()
        N.check(N.lib().wmc_level_create_channel(mesh._h, C.byref(d), level, C.byref(h)))
        self._h = h
        info = N.LevelInfo()
        N.check(N.lib().wmc_level_get_info(self._h, C.byref(info)))
        self.info = _info_dict(info)
        return self

    @property
    def stream(self) -> int:
        return N.lib().wmc_level_stream(self._h) or 0

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            N.lib().wmc_level_destroy(self._h)
            self._h = C.c_void_p()


def eval_pairs(fine: Level, coarse: Level | None, seed: int, level: int, first: int, count: int):
    """Batched sample_delta_q (reference src/mlmc.cpp:21-37) over indices
    first..first+count-1: returns (dq, q_fine, cost dict); QoI vectors
    (info["nq"] > 1) come back with shape (count, nq)."""
    nq = fine.info.get("nq", 1)
    shape = (count,) if nq == 1 else (count, nq)
    dq = np.empty(shape, np.float64)
    qf = np.empty(shape, np.float64)
    cost = N.Cost()
    err = N.Error()
    rc = N.lib().wmc_eval_pairs(fine._h, coarse._h if coarse is not None else None, seed, level, first, count,
                                _dptr(dq), _dptr(qf), C.byref(cost), C.byref(err))
    N.check(rc, err)
    return dq, qf, {k: getattr(cost, k) for k, _ in N.Cost._fields_}


def eval_pairs_device(fine: Level, coarse: Level | None, seed: int, level: int, first: int, count: int,
                      d_dq: int = 0, d_qf: int = 0) -> None:
    """Same work, results left in device memory, no host synchronisation."""
    N.check(N.lib().wmc_eval_pairs_device(fine._h, coarse._h if coarse is not None else None, seed, level, first,
                                          count, d_dq or None, d_qf or None))


def synchronize(level: Level) -> None:
    err = N.Error()
    N.check(N.lib().wmc_synchronize(level._h, C.byref(err)), err)


def kl_modes(sigma: float, corr_len: float, modes: int):
    """The KL expansion's modes for a pointwise evaluator (wmc_kl_modes): [modes, 7]."""
    out = np.empty((modes, 7), np.float64)
    N.check(N.lib().wmc_kl_modes(sigma, corr_len, modes, _dptr(out)))
    return out


def kl_table(cells_x: int, cells_y: int, sigma: float, corr_len: float, modes: int):
    """(table[cell, mode], lambda[mode]) of the log-normal KL field."""
    table = np.empty((cells_x * cells_y, modes), np.float64)
    lam = np.empty(modes, np.float64)
    N.check(N.lib().wmc_kl_table(cells_x, cells_y, sigma, corr_len, modes, _dptr(table), _dptr(lam)))
    return table, lam


def level_draw(level: "Level", seed: int, level_index: int, first: int, count: int) -> np.ndarray:
    """The level's per-sample cell coefficients, shape (count, n_cells)."""
    n_cells = level.spec.cells_x * level.spec.cells_y
    out = np.empty((count, n_cells), np.float64)
    N.check(N.lib().wmc_level_draw(level._h, seed, level_index, first, count, _dptr(out)))
    return out


def level_cfl(level: Level, seed: int, level_index: int, first: int, count: int):
    """Per-sample snapped CFL step and step count as the device computes them."""
    dt = np.zeros(count, np.float64)
    steps = np.zeros(count, np.int64)
    N.check(N.lib().wmc_level_cfl(level._h, seed, level_index, first, count, _dptr(dt),
                                  steps.ctypes.data_as(C.POINTER(C.c_long))))
    return dt, steps


def draw_cells(seed: int, level: int, first: int, count: int, n_cells: int = 16, lo: float = 0.5,
               hi: float = 1.5, device: int = 0) -> np.ndarray:
    out = np.empty((count, n_cells), np.float64)
    N.check(N.lib().wmc_draw_cells(seed, level, first, count, n_cells, lo, hi, device, _dptr(out)))
    return out


def _stats(s: N.LevelStats) -> dict:
    d = {k: getattr(s, k) for k, _ in N.LevelStats._fields_ if k != "cost"}
    d["cost"] = {k: getattr(s.cost, k) for k, _ in N.Cost._fields_}
    return d


def run_mlmc_fixed(levels: list[Level], counts: list[int], seed: int = 0, first: list[int] | None = None) -> list[dict]:
    """Fixed N_l over levels 0..L (BASELINE config 1): per-level LevelAccumulator
    sums and estimators, folded in index order.  With ``first`` the call covers
    indices first[l] .. first[l]+counts[l]-1 (one rank's shard)."""
    n = len(levels)
    arr = (C.c_void_p * n)(*[lv._h.value for lv in levels])
    cnt = (C.c_long * n)(*counts)
    fst = (C.c_long * n)(*(first or [0] * n))
    stats = (N.LevelStats * n)()
    err = N.Error()
    N.check(N.lib().wmc_run_mlmc_fixed(arr, n, fst, cnt, seed, stats, C.byref(err)), err)
    return [_stats(stats[i]) for i in range(n)]


@dataclass
class MlmcConfig:
    """Reference MlmcConfig (include/wavemc/mlmc.hpp:14-23)."""
    eps: float = 1e-3
    alpha: float = 2.0
    initial_samples: int = 16
    initial_levels: int = 2
    max_level: int = 6
    master_seed: int = 0
    bias_window: int = 1


@dataclass
class MlmcResult:
    estimate: float
    converged: bool
    levels_used: int
    total_variance: float
    bias: float
    total_model_cost: float
    rmse: float
    levels: list = field(default_factory=list)
    estimate_vector: object = None  # QoI vectors: the estimate per output (numpy array)


def run_mlmc(levels: list[Level], model_cost: list[float], config: MlmcConfig | None = None) -> MlmcResult:
    """Adaptive Giles driver (reference run_mlmc, src/mlmc.cpp:165-233)."""
    config = config or MlmcConfig()
    n = len(levels)
    arr = (C.c_void_p * n)(*[lv._h.value for lv in levels])
    cost = (C.c_double * n)(*model_cost)
    cfg = N.MlmcConfig(config.eps, config.alpha, config.initial_samples, config.initial_levels, config.max_level,
                       config.master_seed, config.bias_window)
    res = N.MlmcResult()
    stats = (N.LevelStats * n)()
    err = N.Error()
    est = np.zeros(max(1, levels[0].info.get("nq", 1)), np.float64)
    N.check(N.lib().wmc_run_mlmc_vec(arr, n, cost, C.byref(cfg), C.byref(res), stats, _dptr(est), C.byref(err)), err)
    return MlmcResult(res.estimate, bool(res.converged), res.levels_used, res.total_variance, res.bias,
                      res.total_model_cost, res.rmse, [_stats(stats[i]) for i in range(res.levels_used + 1)], est)


def _groups(level_groups: list[list[Level]]):
    n_dev, n = len(level_groups), len(level_groups[0])
    if any(len(g) != n for g in level_groups):
        raise ValueError("every device group needs the same number of levels")
    arr = (C.c_void_p * (n_dev * n))(*[lv._h.value for g in level_groups for lv in g])
    return arr, n_dev, n


def run_mlmc_fixed_multi(level_groups: list[list[Level]], counts: list[int], seed: int = 0) -> list[dict]:
    """run_mlmc_fixed over several devices (wmc_run_mlmc_fixed_multi): one
    level list per device, 64-sample granules per device, one host thread per
    device, host fold in index order -- bitwise the one-device result."""
    arr, n_dev, n = _groups(level_groups)
    cnt = (C.c_long * n)(*counts)
    stats = (N.LevelStats * n)()
    err = N.Error()
    N.check(N.lib().wmc_run_mlmc_fixed_multi(arr, n_dev, n, cnt, seed, stats, C.byref(err)), err)
    return [_stats(stats[i]) for i in range(n)]


def run_mlmc_multi(level_groups: list[list[Level]], model_cost: list[float],
                   config: MlmcConfig | None = None) -> MlmcResult:
    """The adaptive driver over several devices (wmc_run_mlmc_multi)."""
    config = config or MlmcConfig()
    arr, n_dev, n = _groups(level_groups)
    cost = (C.c_double * n)(*model_cost)
    cfg = N.MlmcConfig(config.eps, config.alpha, config.initial_samples, config.initial_levels, config.max_level,
                       config.master_seed, config.bias_window)
    res = N.MlmcResult()
    stats = (N.LevelStats * n)()
    err = N.Error()
    est = np.zeros(max(1, level_groups[0][0].info.get("nq", 1)), np.float64)
    N.check(N.lib().wmc_run_mlmc_multi(arr, n_dev, n, cost, C.byref(cfg), C.byref(res), stats, _dptr(est),
                                       C.byref(err)), err)
    return MlmcResult(res.estimate, bool(res.converged), res.levels_used, res.total_variance, res.bias,
                      res.total_model_cost, res.rmse, [_stats(stats[i]) for i in range(res.levels_used + 1)], est)


def optimal_samples(variances, costs, eps: float, min_samples: int = 2) -> list[int]:
    """Reference optimal_samples (src/mlmc.cpp:75-92)."""
    n = len(variances)
    v = (C.c_double * n)(*variances)
    c = (C.c_double * n)(*costs)
    out = (C.c_long * n)()
    N.check(N.lib().wmc_optimal_samples(v, c, n, eps, min_samples, out))
    return list(out)


def bias_proxy_sq(mean_dq: float, alpha: float = 2.0) -> float:
    """Reference bias_proxy_sq (src/mlmc.cpp:94-98) on the scalar QoI."""
    return N.lib().wmc_bias_proxy_sq(mean_dq, alpha)


def moments_device(level: Level, d_dq: int, d_q: int, count: int, d_out: int) -> None:
    """d_out[0..3] += {sum dq, sum dq^2, sum q, sum q^2} on the device."""
    N.check(N.lib().wmc_moments_device(level._h, d_dq, d_q, count, d_out))


def profile_enable(level: Level, on: bool = True) -> None:
    N.check(N.lib().wmc_profile_enable(level._h, int(on)))


def profile_read(level: Level) -> dict:
    sm, su, sr = C.c_double(), C.c_double(), C.c_double()
    ns, nu, nr = C.c_long(), C.c_long(), C.c_long()
    N.check(N.lib().wmc_profile_read(level._h, C.byref(sm), C.byref(ns), C.byref(su), C.byref(nu), C.byref(sr),
                                     C.byref(nr)))
    return {"sweep_ms": sm.value, "sweep_launches": ns.value, "sub_ms": su.value, "sub_launches": nu.value,
            "upd_ms": sr.value, "upd_launches": nr.value}


def launch_count() -> int:
    return N.lib().wmc_launch_count()


def device_count() -> int:
    return N.lib().wmc_device_count()
