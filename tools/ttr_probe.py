"""Time-to-RMSE of the adaptive driver (wmc_run_mlmc) on the config-1 (and,
with --kl, config-4) hierarchy: wall time around the public call, after one
warm-up run at a looser target.  python tools/ttr_probe.py [--eps E] [--kl]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_11117_b200 import configs, wavemc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--kl", action="store_true")
    ap.add_argument("--repeat", type=int, default=3)
    a = ap.parse_args()
    levels = [configs.build_level(d, kl=a.kl) for d in configs.config1()]
    costs = [lv.info["dof_updates_per_solve"] for lv in levels]
    wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=a.eps * 4))
    for _ in range(a.repeat):
        t0 = time.perf_counter()
        r = wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=a.eps))
        dt = time.perf_counter() - t0
        print(f"eps={a.eps} kl={a.kl} seconds={dt:.4f} N_l={[s['n_samples'] for s in r.levels]} "
              f"estimate={r.estimate!r} rmse={r.rmse:.3e}")


if __name__ == "__main__":
    main()
