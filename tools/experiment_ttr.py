"""Time-to-RMSE of the reference's own 1D experiments on the device: the
adaptive driver over levels 0..4 at the given eps (wall time around the
public call, after a warm-up at 4 eps).  python tools/experiment_ttr.py smooth1d lts 1e-3"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_11117_b200 import wavemc  # noqa: E402
from paper_2106_11117_b200._native import WMC_LEAPFROG, WMC_LOCAL_TIME_STEPPING  # noqa: E402


def main():
    name, kind, eps = sys.argv[1], sys.argv[2], float(sys.argv[3])
    integ = WMC_LOCAL_TIME_STEPPING if kind == "lts" else WMC_LEAPFROG
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "mesh1d",
                           f"{name}_L4.json")) as f:  # the reference's build_hierarchy meshes
        meshes = wavemc.Mesh1D.hierarchy(json.load(f)["levels"])
    levels = [wavemc.Level.experiment(name, l, meshes[l], integ) for l in range(5)]
    cost = wavemc.experiment_model_cost(name, integ)
    wavemc.run_mlmc(levels, cost, wavemc.MlmcConfig(eps=4 * eps, max_level=4))
    for _ in range(2):
        t0 = time.perf_counter()
        r = wavemc.run_mlmc(levels, cost, wavemc.MlmcConfig(eps=eps, max_level=4))
        print(f"{name} {kind} eps={eps} seconds={time.perf_counter() - t0:.4f} "
              f"N_l={[s['n_samples'] for s in r.levels]} estimate_norm={r.estimate!r} converged={r.converged}")


if __name__ == "__main__":
    main()
