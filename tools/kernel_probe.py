"""Run one config-1 level (fine solves only) for a few batches: the small,
repeatable command profiled with ncu (see profiles/README.md)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_11117_b200 import configs, wavemc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--count", type=int, default=1184)
    ap.add_argument("--generic", action="store_true", help="mesh without lattice metadata")
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--square", type=int, nargs=2, metavar=("N_COARSE", "RATIO"),
                    help="custom refined-square mesh (LTS with p = RATIO, dt = 0.2 h)")
    ap.add_argument("--steps", type=int, default=0, help="limit the horizon to this many global steps")
    ap.add_argument("--nocheck", action="store_true", help="device-resident results, no instability check")
    ap.add_argument("--profile", action="store_true", help="per-kernel CUDA-event times of the last repeat")
    ap.add_argument("--p", type=int, default=0, help="override the number of substeps (timing studies)")
    ap.add_argument("--config2", action="store_true", help="config-2 level (graded L-shape, nested tiers)")
    a = ap.parse_args()
    d = (configs.config2() if a.config2 else configs.config1())[a.level]
    if a.square:
        nc, r = a.square
        d = configs.LevelDef(nc, r, 0.2 / nc, r, d.integrator)
    if a.steps:
        d = configs.LevelDef(d.n_coarse, d.ratio, d.dt, d.substeps, d.integrator, final_time=a.steps * d.dt,
                             shape=d.shape, tiers=d.tiers)
    if a.p:
        d = configs.LevelDef(d.n_coarse, d.ratio, d.dt, a.p, d.integrator, final_time=d.final_time)
    m = configs.build_mesh(d)
    if a.generic:
        m = wavemc.Mesh.from_arrays(*m.arrays())
    lv = wavemc.Level(m, configs.level_spec(d))
    if a.nocheck:
        import torch
        dq_t = torch.empty(a.count, dtype=torch.float64, device="cuda")
        qf_t = torch.empty(a.count, dtype=torch.float64, device="cuda")
    for r in range(a.repeat):
        if a.profile and r == a.repeat - 1:
            wavemc.profile_enable(lv, True)
        t0 = time.perf_counter()
        if a.nocheck:
            wavemc.eval_pairs_device(lv, None, 0, a.level, 0, a.count, dq_t.data_ptr(), qf_t.data_ptr())
            wavemc.synchronize(lv)
            q = qf_t.cpu().numpy()
        else:
            _, q, _ = wavemc.eval_pairs(lv, None, 0, a.level, 0, a.count)
        dt = time.perf_counter() - t0
        upd = a.count * lv.info["dof_updates_per_solve"]
        if a.profile and r == a.repeat - 1:
            print("profile", wavemc.profile_read(lv))
        print(f"level {a.level} path={lv.info['substep_path']} fused={lv.info['fused']} n={lv.info['n']} n_r={lv.info['n_r']} "
              f"{a.count} solves {dt:.3f} s "
              f"{upd / dt:.3e} DOF-updates/s q0={q[0]:.12e}")


if __name__ == "__main__":
    main()
