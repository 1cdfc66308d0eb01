"""ctypes binding of the C ABI in include/wavemc_b200.h.

The product path has no fallback: if libwavemc_b200.so is missing or fails to
load, every call raises.  Build it with ``python -c 'import __graft_entry__ as
g; g.build()'`` (or ``make -C paper_2106_11117_b200/csrc``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WMC_LIB_PATH") or os.path.join(_HERE, "libwavemc_b200.so")  # override: tuning builds

WMC_OK = 0
WMC_CONFIG_ERROR = 2
WMC_NUMERICAL_ERROR = 3
WMC_DEVICE_ERROR = 4
WMC_LEAPFROG = 0
WMC_LOCAL_TIME_STEPPING = 1
WMC_FIELD_UNIFORM = 0
WMC_FIELD_LOGNORMAL_KL = 1
WMC_FIELD_LOGNORMAL_KL_ELEMENT = 2


class SquareMeshSpec(C.Structure):
    _fields_ = [("n_coarse", C.c_int), ("ratio", C.c_int), ("fine_lo", C.c_double), ("fine_hi", C.c_double),
                ("snap", C.c_double), ("small_factor", C.c_double)]


class LevelDesc(C.Structure):
    _fields_ = [("cells_x", C.c_int), ("cells_y", C.c_int), ("coef_lo", C.c_double), ("coef_hi", C.c_double),
                ("final_time", C.c_double), ("dt", C.c_double), ("substeps", C.c_int), ("nu", C.c_double),
                ("integrator", C.c_int), ("ic_x", C.c_double), ("ic_y", C.c_double), ("ic_width2", C.c_double),
                ("qoi_box", C.c_double * 4), ("device", C.c_int), ("batch", C.c_int), ("field", C.c_int),
                ("kl_sigma", C.c_double), ("kl_corr_len", C.c_double), ("kl_modes", C.c_int),
                ("tiers", C.c_int), ("domain", C.c_double * 4), ("qoi_mean", C.c_int),
                ("cfl_safety", C.c_double)]


WMC_EXP_SMOOTH1D = 1
WMC_EXP_JUMP1D = 2
WMC_EXP_CHANNEL2D = 3


class ExperimentDesc(C.Structure):
    _fields_ = [("experiment", C.c_int), ("integrator", C.c_int), ("h0", C.c_double), ("fine_h", C.c_double),
                ("final_time", C.c_double), ("nu", C.c_double), ("safety", C.c_double), ("grid_n", C.c_int),
                ("max_level", C.c_int), ("device", C.c_int), ("batch", C.c_int)]


class LShapeMeshSpec(C.Structure):
    _fields_ = [("n_per_unit", C.c_int), ("tiers", C.c_int), ("grade_radius", C.c_double)]


class LevelInfo(C.Structure):
    _fields_ = [("n", C.c_int), ("n_r", C.c_int), ("n_p", C.c_int), ("p", C.c_int), ("n_steps", C.c_long),
                ("dt", C.c_double), ("nnz", C.c_long), ("ap_nnz", C.c_long), ("n_recipes", C.c_long),
                ("batch", C.c_int), ("dof_updates_per_solve", C.c_double), ("lattice", C.c_int),
                ("substep_path", C.c_int), ("tiers", C.c_int), ("n_r_tier", C.c_int * 8),
                ("n_structured", C.c_long), ("nq", C.c_int), ("fused", C.c_int)]


class TilePlanInfo(C.Structure):
    _fields_ = [("ok", C.c_int), ("n_tiles", C.c_int), ("n_slabs", C.c_int), ("max_gen", C.c_int),
                ("work_factor", C.c_double), ("streamed_frac", C.c_double), ("layout", C.c_char * 32),
                ("reason", C.c_char * 256)]


class Cost(C.Structure):
    _fields_ = [("matvec_full", C.c_long), ("matvec_fine", C.c_long), ("matvec_coarse", C.c_long),
                ("weighted_work", C.c_long), ("dof_updates", C.c_double)]


class Error(C.Structure):
    _fields_ = [("sample", C.c_long), ("step", C.c_long), ("level", C.c_int)]


class LevelStats(C.Structure):
    _fields_ = [("level", C.c_int), ("n_samples", C.c_long), ("sum_dq", C.c_double), ("sum_dq2", C.c_double),
                ("sum_q", C.c_double), ("sum_q2", C.c_double), ("variance", C.c_double),
                ("mc_variance", C.c_double), ("mean_dq", C.c_double), ("model_cost", C.c_double), ("cost", Cost)]


class MlmcConfig(C.Structure):
    _fields_ = [("eps", C.c_double), ("alpha", C.c_double), ("initial_samples", C.c_int),
                ("initial_levels", C.c_int), ("max_level", C.c_int), ("master_seed", C.c_uint64),
                ("bias_window", C.c_int)]


class MlmcResult(C.Structure):
    _fields_ = [("estimate", C.c_double), ("converged", C.c_int), ("levels_used", C.c_int),
                ("total_variance", C.c_double), ("bias", C.c_double), ("total_model_cost", C.c_double),
                ("rmse", C.c_double)]


P = C.POINTER
_VP = C.c_void_p
_DP = P(C.c_double)

# (name, restype, argtypes) for every symbol include/wavemc_b200.h declares
SIGNATURES = [
    ("wmc_mesh_build_square", C.c_int, [P(SquareMeshSpec), P(_VP)]),
    ("wmc_mesh_build_lshape", C.c_int, [P(LShapeMeshSpec), P(_VP)]),
    ("wmc_mesh_create", C.c_int, [C.c_int, C.c_int, _DP, P(C.c_int), P(C.c_ubyte), P(C.c_ubyte), C.c_double,
                                  C.c_double, P(_VP)]),
    ("wmc_mesh_info", C.c_int, [_VP, P(C.c_int), P(C.c_int), _DP, _DP]),
    ("wmc_mesh_export", C.c_int, [_VP, _DP, P(C.c_int), P(C.c_ubyte), P(C.c_ubyte)]),
    ("wmc_mesh_dump", C.c_int, [_VP, C.c_char_p]),
    ("wmc_mesh_destroy", None, [_VP]),
    ("wmc_level_desc_default", None, [P(LevelDesc)]),
    ("wmc_level_create", C.c_int, [_VP, P(LevelDesc), P(_VP)]),
    ("wmc_experiment_desc_default", None, [P(ExperimentDesc), C.c_int]),
    ("wmc_mesh1d_create", C.c_int, [C.c_int, _DP, P(C.c_ubyte), C.c_double, C.c_double, P(_VP)]),
    ("wmc_mesh1d_destroy", None, [_VP]),
    ("wmc_level_create_experiment", C.c_int, [_VP, C.c_int, P(ExperimentDesc), C.c_int, P(_VP)]),
    ("wmc_experiment_plan", C.c_int, [_VP, C.c_int, P(ExperimentDesc), C.c_int, P(LevelInfo)]),
    ("wmc_level_create_channel", C.c_int, [_VP, P(ExperimentDesc), C.c_int, P(_VP)]),
    ("wmc_channel_plan", C.c_int, [_VP, P(ExperimentDesc), C.c_int, P(LevelInfo)]),
    ("wmc_experiment_model_cost", C.c_double, [P(ExperimentDesc), C.c_int]),
    ("wmc_level_plan", C.c_int, [_VP, P(LevelDesc), P(LevelInfo)]),
    ("wmc_tile_plan", C.c_int, [_VP, P(LevelDesc), C.c_int, P(TilePlanInfo)]),
    ("wmc_level_get_info", C.c_int, [_VP, P(LevelInfo)]),
    ("wmc_level_destroy", None, [_VP]),
    ("wmc_eval_pairs", C.c_int, [_VP, _VP, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, _DP, _DP, P(Cost),
                                 P(Error)]),
    ("wmc_eval_pairs_device", C.c_int, [_VP, _VP, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, _VP, _VP]),
    ("wmc_level_stream", _VP, [_VP]),
    ("wmc_synchronize", C.c_int, [_VP, P(Error)]),
    ("wmc_kl_table", C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _DP, _DP]),
    ("wmc_kl_modes", C.c_int, [C.c_double, C.c_double, C.c_int, _DP]),
    ("wmc_level_draw", C.c_int, [_VP, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, _DP]),
    ("wmc_level_cfl", C.c_int, [_VP, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, P(C.c_double), P(C.c_long)]),
    ("wmc_draw_cells", C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                 C.c_int, _DP]),
    ("wmc_run_mlmc_fixed", C.c_int, [P(_VP), C.c_int, P(C.c_long), P(C.c_long), C.c_uint64, P(LevelStats),
                                     P(Error)]),
    ("wmc_mlmc_config_default", None, [P(MlmcConfig)]),
    ("wmc_run_mlmc", C.c_int, [P(_VP), C.c_int, _DP, P(MlmcConfig), P(MlmcResult), P(LevelStats), P(Error)]),
    ("wmc_run_mlmc_vec", C.c_int, [P(_VP), C.c_int, _DP, P(MlmcConfig), P(MlmcResult), P(LevelStats), _DP,
                                   P(Error)]),
    ("wmc_run_mlmc_fixed_multi", C.c_int, [P(_VP), C.c_int, C.c_int, P(C.c_long), C.c_uint64, P(LevelStats),
                                           P(Error)]),
    ("wmc_run_mlmc_multi", C.c_int, [P(_VP), C.c_int, C.c_int, _DP, P(MlmcConfig), P(MlmcResult), P(LevelStats), _DP,
                                     P(Error)]),
    ("wmc_optimal_samples", C.c_int, [_DP, _DP, C.c_int, C.c_double, C.c_long, P(C.c_long)]),
    ("wmc_bias_proxy_sq", C.c_double, [C.c_double, C.c_double]),
    ("wmc_moments_device", C.c_int, [_VP, _VP, _VP, C.c_uint64, _VP]),
    ("wmc_profile_enable", C.c_int, [_VP, C.c_int]),
    ("wmc_profile_read", C.c_int, [_VP, _DP, P(C.c_long), _DP, P(C.c_long), _DP, P(C.c_long)]),
    ("wmc_launch_count", C.c_long, []),
    ("wmc_last_error", C.c_char_p, []),
    ("wmc_device_count", C.c_int, []),
]

_lib = None


def lib():
    """Load libwavemc_b200.so (raises if it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"wavemc-b200: native library {LIB_PATH} is not built "
                               "(run __graft_entry__.build()); there is no CPU fallback")
        handle = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


class WavemcError(RuntimeError):
    def __init__(self, code: int, message: str, sample: int = -1, step: int = 0, level: int = -1):
        super().__init__(message)
        self.code = code
        self.sample = sample
        self.step = step
        self.level = level


class ConfigError(WavemcError):
    pass


class NumericalError(WavemcError):
    pass


class DeviceError(WavemcError):
    pass


def check(code: int, err: Error | None = None) -> None:
    if code == WMC_OK:
        return
    msg = (lib().wmc_last_error() or b"").decode()
    cls = {WMC_CONFIG_ERROR: ConfigError, WMC_NUMERICAL_ERROR: NumericalError}.get(code, DeviceError)
    if err is not None:
        raise cls(code, msg, err.sample, err.step, err.level)
    raise cls(code, msg)
