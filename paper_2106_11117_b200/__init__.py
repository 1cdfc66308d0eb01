"""wavemc-b200: B200-native batched LF / LF-LTS wave-sample evaluation for
MLMC (arXiv 2106.11117).  See DESIGN.md."""
from .wavemc import (ConfigError, DeviceError, Level, LevelSpec, Mesh, MlmcConfig, MlmcResult,  # noqa: F401
                     NumericalError, WavemcError, device_count, draw_cells, eval_pairs, eval_pairs_device,
                     run_mlmc, run_mlmc_fixed, synchronize)

__all__ = ["Mesh", "Level", "LevelSpec", "eval_pairs", "eval_pairs_device", "run_mlmc", "run_mlmc_fixed",
           "MlmcConfig", "MlmcResult", "draw_cells", "synchronize", "device_count", "WavemcError", "ConfigError",
           "NumericalError", "DeviceError"]
