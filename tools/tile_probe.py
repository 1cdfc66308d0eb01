"""Config-3 probe of the tiled step (profiling helper): one batch of the
config-3 level with a short horizon, timed with CUDA events per path.

  python tools/tile_probe.py [--steps N] [--count C] [--path tiled|global]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2106_11117_b200 import configs, wavemc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--count", type=int, default=256)
    ap.add_argument("--path", default="tiled")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    if args.path == "global":
        os.environ["WMC_TILED"] = "0"
    d = configs.config3()
    t0 = time.time()
    mesh = configs.build_mesh(d)
    spec = wavemc.LevelSpec(dt=d.dt, substeps=d.substeps, final_time=args.steps * d.dt, batch=args.count)
    lv = wavemc.Level(mesh, spec)
    print(f"setup {time.time() - t0:.1f} s, path {lv.info['substep_path']}, batch {lv.info['batch']}", flush=True)
    dq = torch.empty(args.count, dtype=torch.float64, device="cuda")
    qf = torch.empty(args.count, dtype=torch.float64, device="cuda")
    wavemc.profile_enable(lv, True)
    for r in range(args.reps):
        wavemc.eval_pairs_device(lv, None, 0, 0, 0, args.count, dq.data_ptr(), qf.data_ptr())
        wavemc.synchronize(lv)
        p = wavemc.profile_read(lv)
        upd = lv.info["dof_updates_per_solve"] * args.count
        per_step = p["sub_ms"] / max(1, p["sub_launches"])
        print(f"rep {r}: sweep {p['sweep_ms']:.2f} ms / {p['sweep_launches']}, substep {p['sub_ms']:.2f} ms / "
              f"{p['sub_launches']} ({per_step:.3f} ms per step), total DOF-upd/s "
              f"{upd / ((p['sweep_ms'] + p['sub_ms']) * 1e-3):.3e}", flush=True)


if __name__ == "__main__":
    main()
