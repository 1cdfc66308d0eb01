"""Inputs of the reference CPU arm (bench.py --impl reference, the CPU legs):
the BASELINE config's meshes in the reference's fixture format plus the
level data the arm needs (dt, p, DOF-updates per solve), written by this
separate process so the timed reference process never maps the product
library.  Meshes come from the shared problem definition (the same builder
the device path uses, so geometry is never a parity variable).

  python tools/dump_inputs.py --config C --out DIR [--final-time T] [--lf] [--kl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2106_11117_b200 import configs, wavemc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--final-time", type=float, default=None)
    ap.add_argument("--lf", action="store_true", help="config 1: the global leap-frog arm (dt = 0.2 h_min)")
    ap.add_argument("--kl", action="store_true", help="config 4: write the log-normal KL table too")
    ap.add_argument("--kl-element", action="store_true",
                    help="config 4: the field at the element centroids (the KL mode list instead of the cell table)")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    if a.config == 0:
        defs = [configs.config0()]
    elif a.config == 2:
        defs = configs.config2()
    elif a.config == 3:
        defs = [configs.config3()]
    else:
        defs = configs.config1("lf" if a.lf else "lts")
    levels = []
    for l, d in enumerate(defs):
        path = os.path.join(a.out, f"l{l}.mesh")
        mesh = configs.build_mesh(d)
        mesh.dump(path)
        spec = configs.level_spec(d)
        if a.final_time is not None:
            spec.final_time = a.final_time
        plan = wavemc.level_plan(mesh, spec)
        levels.append({"mesh": path, "dt": d.dt, "p": d.substeps, "tiers": d.tiers,
                       "dof_updates_per_solve": plan["dof_updates_per_solve"], "n": plan["n"], "n_r": plan["n_r"],
                       "n_steps": plan["n_steps"]})
    out = {"config": a.config, "levels": levels}
    if a.kl:
        kl = configs.KL_FIELD
        table, _ = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
        path = os.path.join(a.out, "kl.txt")
        with open(path, "w") as f:
            f.write(f"{table.shape[0]} {table.shape[1]}\n")
            f.write("\n".join(repr(float(v)) for v in table.ravel()) + "\n")
        out["kl"] = {"kl-table": path, "cells-x": kl["cells"][0], "cells-y": kl["cells"][1]}
        if a.kl_element:
            modes = wavemc.kl_modes(kl["sigma"], kl["corr_len"], kl["modes"])
            mpath = os.path.join(a.out, "kl_modes.txt")
            with open(mpath, "w") as f:
                f.write(f"{modes.shape[0]}\n")
                f.write("\n".join(repr(float(v)) for v in modes.ravel()) + "\n")
            out["kl"] = {"kl-modes": mpath}
    with open(os.path.join(a.out, "inputs.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
