#!/usr/bin/env python
"""Benchmark of the batched LF-LTS MLMC hot path (BASELINE.json config 1).

One step = the whole fixed-N MLMC estimator of config 1: coupled pairs on
levels 0..4 (h_l = 1/16..1/256, p_l = 32..2, N_l = 65536, 16384, 4096, 1024,
256), both solves of every pair, FP64, plus the per-level moment sums and
(N > 1) one NCCL allreduce of them.  Metric: DOF-updates/s with
U = n + (p-1)|R| per global step per solve.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun every rank evaluates the index range [r N_l / G, (r+1) N_l / G)
of every level (weak in samples per GPU? no: total work is fixed -> "strong").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

METRIC = "DOF-updates/s (FP64, LTS substeps incl.)"
TTR_EPS = 1e-4  # RMSE target of the time-to-RMSE run (config-1 hierarchy)
UNIT = "DOF-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=float, default=None,
                    help="fraction of N_l (default 1.0 = the BASELINE counts; config 3: 0.03, a 246-sample slice "
                         "of the 8192 -- per-sample cost is uniform, the full set is ~20 min per step)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4],
                    help="BASELINE config: 1 (default, MLMC), 0 (single-level MC), 2 (graded L-shape MLMC, "
                         "nested 3-tier LTS), 3 (large single level), 4 (adaptive MLMC to an RMSE target, "
                         "log-normal KL coefficient)")
    ap.add_argument("--eps", type=float, default=None, help="config 4: RMSE target (default BASELINE 1e-3)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        exe = shutil.which("nvidia-smi")
        if not exe:
            return
        while not self._stop.is_set():
            try:
                out = subprocess.run([exe, "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baselines (the reference compiled from its own sources, else our port)

def workload(config: int):
    """(level defs, N per level, description, CPU horizon override)."""
    from paper_2106_11117_b200 import configs
    if config == 0:
        return [configs.config0()], [configs.CONFIG0_COUNT], "BASELINE config 0: single-level MC, h=1/32 refined x4, p=4", None
    if config == 2:
        defs = configs.config2()
        # the CPU sample keeps every level but shortens the horizon to T/8
        return defs, list(configs.CONFIG2_COUNTS), (
            "BASELINE config 2: graded L-shape MLMC, nested LTS 3 tiers x p=2, 5 levels h=1/16..1/256, T=2"), 0.25
    if config == 3:
        d = configs.config3()
        # the CPU sample keeps the mesh and the per-step work but shortens the
        # horizon to 16 global steps (per-step cost is uniform in time)
        return [d], [configs.CONFIG3_COUNT], "BASELINE config 3: single level h=1/1024 refined x8, p=8, T=0.5", 16 * d.dt
    return configs.config1(), list(configs.CONFIG1_COUNTS), (
        "BASELINE config 1: fixed-N MLMC, LF-LTS, 5 levels h=1/16..1/256, p=32..2"), None


def oracle_problem(d, final_time=None):
    """The C restatement's problem for a level definition (test-side mirror of
    configs.level_spec)."""
    import oracle_py
    from paper_2106_11117_b200 import configs
    T = d.final_time if final_time is None else final_time
    if d.shape == "lshape":
        c = configs.CONFIG2_PROBLEM
        return oracle_py.problem(d.dt, d.substeps, final_time=T, cells=c["cells"], ic=c["ic"], box=c["qoi_box"],
                                 domain=c["domain"], qoi_mean=True, tiers=d.tiers)
    return oracle_py.problem(d.dt, d.substeps, final_time=T)


def ref_sample_counts(threads: int, defs=None):
    """Bounded sample of config 1 for the CPU, in the proportions of N_l
    (65536 : 16384 : 4096 : 1024 : 256 = 256 : 64 : 16 : 4 : 1), sized for
    ~10-15 s of wall time on `threads` cores (measured: 2.8 s for a quarter of
    this sample on 16 cores)."""
    t = max(1, threads)
    if defs is not None and defs[0].shape == "lshape":  # config 2: N_l halving, horizon T/8
        return [8 * t, 4 * t, 2 * t, t, max(1, t // 2)]
    return [64 * t, 16 * t, 4 * t, t, max(1, t // 4)]


def run_reference_cpu(defs, threads: int, final_time=None):
    """A bounded sample through the unmodified reference library (oracle/_ref),
    its own run_jobs-style pool of `threads` workers.  Returns dict."""
    import oracle_py
    from paper_2106_11117_b200 import configs
    counts = ref_sample_counts(threads, defs) if len(defs) > 1 else [4 * threads if final_time is None else threads]
    tmp = tempfile.mkdtemp(prefix="wmc_bench_")
    specs = []
    nested = any(d.tiers > 1 for d in defs)
    for l, d in enumerate(defs):
        p = os.path.join(tmp, f"l{l}.mesh")
        configs.build_mesh(d).dump(p)
        # config 2: the reference has no nested tiers; its own LF-LTS on the
        # same mesh needs P = P_1 and p = 2^tiers (stable at the finest tier)
        specs.append((p, d.dt, d.substeps ** d.tiers if nested else d.substeps))
    drv = oracle_py.RefDriver()
    extra = {"T": repr(final_time)} if final_time is not None else {}
    if nested:
        c = configs.CONFIG2_PROBLEM
        extra.update({"T": repr(final_time if final_time is not None else defs[0].final_time),
                      "cells-x": c["cells"][0], "cells-y": c["cells"][1], "ic": ",".join(map(repr, c["ic"])),
                      "box": ",".join(map(repr, c["qoi_box"])), "domain": ",".join(map(repr, c["domain"])),
                      "qoi-mean": 1})
    res = drv.mlmc(specs, counts, threads=threads, **extra)
    shutil.rmtree(tmp, ignore_errors=True)
    work = res["dof_updates"]
    if nested:  # the same samples counted in the config-2 (nested) units
        from paper_2106_11117_b200 import wavemc
        upd = []
        for d in defs:
            spec = configs.level_spec(d)
            if final_time is not None:
                spec.final_time = final_time
            upd.append(wavemc.level_plan(configs.build_mesh(d), spec)["dof_updates_per_solve"])
        work = sum(n * (upd[l] + (upd[l - 1] if l else 0.0)) for l, n in enumerate(counts))
    return {"value": work / res["seconds"], "seconds": res["seconds"], "dof_updates": work, "counts": counts,
            "kind": "reference", "cores": res["threads"],
            "note": ("reference single-tier LF-LTS (P = P_1, p = 8) on the config-2 meshes and samples (it has no "
                     "nested tiers); value = nested-scheme DOF-updates of the same samples / reference time"
                     if nested else None)}


def run_port_cpu(defs, threads: int, final_time=None):
    """Fallback when oracle/_ref is absent: our C restatement, `threads` workers."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle_py
    from paper_2106_11117_b200 import configs
    oracle_py.build()
    orc = oracle_py.COracle()
    counts = ref_sample_counts(threads, defs) if len(defs) > 1 else [4 * threads if final_time is None else threads]
    from paper_2106_11117_b200 import wavemc
    meshes = [oracle_py.MeshArrays(*configs.build_mesh(d).arrays()) for d in defs]
    T = [final_time if final_time is not None else d.final_time for d in defs]
    probs = [oracle_problem(d, t) for d, t in zip(defs, T)]
    upd = []
    for d, t in zip(defs, T):
        spec = configs.level_spec(d)
        spec.final_time = t
        upd.append(wavemc.level_plan(configs.build_mesh(d), spec)["dof_updates_per_solve"])
    jobs = [(l, i) for l in range(len(defs)) for i in range(counts[l])]

    def one(job):
        l, i = job
        rc, _, _, _, _ = orc.eval_pairs(meshes[l], probs[l], meshes[l - 1] if l else None,
                                        probs[l - 1] if l else None, 0, l, i, 1)
        return upd[l] + (upd[l - 1] if l else 0.0)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        total = sum(ex.map(one, jobs))
    dt = time.perf_counter() - t0
    return {"value": total / dt, "seconds": dt, "dof_updates": total, "counts": counts, "kind": "port",
            "cores": threads}


def reference_time_to_rmse(defs, threads: int):
    """The reference's own run_mlmc (src/mlmc.cpp:165-233) to RMSE TTR_EPS on
    the config-1 hierarchy, wall time measured by the driver."""
    import oracle_py
    from paper_2106_11117_b200 import configs
    tmp = tempfile.mkdtemp(prefix="wmc_ttr_")
    specs = []
    for l, d in enumerate(defs):
        p = os.path.join(tmp, f"l{l}.mesh")
        configs.build_mesh(d).dump(p)
        specs.append((p, d.dt, d.substeps))
    res = oracle_py.RefDriver().adaptive(specs, TTR_EPS, threads=threads)
    shutil.rmtree(tmp, ignore_errors=True)
    return {"eps": TTR_EPS, "seconds": res["seconds"], "rmse": math.sqrt(res["total_variance"] + res["bias"]),
            "converged": res["converged"], "estimate": res["estimate"], "N_l": [lv["N"] for lv in res["levels"]],
            "threads": res["threads"]}


def cpu_baseline(defs, threads: int, final_time=None):
    import oracle_py
    if os.path.exists(oracle_py.REF_DRIVER):
        return run_reference_cpu(defs, threads, final_time)
    return run_port_cpu(defs, threads, final_time)


# ---------------------------------------------------------------------------

def reference_arm(args, world, rank):
    from paper_2106_11117_b200 import configs
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    defs, counts_total, label, cpu_T = workload(args.config)
    try:
        runs = [cpu_baseline(defs, threads, cpu_T) for _ in range(args.warmup + args.steps)]
    except Exception as exc:  # the oracle always exists; report loudly
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU run failed: {exc}"}))
        return 0
    timed = runs[args.warmup:]
    value = sum(r["dof_updates"] for r in timed) / sum(r["seconds"] for r in timed)
    ttr = None
    if args.config == 1:
        try:
            ttr = reference_time_to_rmse(defs, threads)
        except Exception as exc:
            ttr = {"eps": TTR_EPS, "error": str(exc)}
    r0 = timed[0]
    sample = (f"config {args.config} bounded sample N_l={r0['counts']} (of {counts_total}) per step"
              + (f", horizon shortened to T={cpu_T!r}" if cpu_T is not None else "")
              + f", {r0['cores']} threads, {r0['kind']}"
              + (f"; {r0['note']}" if r0.get("note") else ""))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(r["seconds"] for r in timed) / len(timed),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based RNG draws, seed 0)",
            "config": {"workload": label + " (bounded CPU sample)",
                       "parallelism": f"{r0['cores']} CPU threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r0["cores"], "kind": r0["kind"],
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "time_to_rmse": ttr}
    print(json.dumps(line))
    return 0


def b200_arm(args, world, rank, local):
    import torch

    from paper_2106_11117_b200 import configs, shard, wavemc

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    defs, counts_total, label, cpu_T = workload(args.config)
    if args.scale is None:
        args.scale = 0.03 if args.config == 3 else 1.0
    if args.scale != 1.0:
        label += f" (N_l scaled by {args.scale})"
    counts_total = [max(1, int(round(n * args.scale))) for n in counts_total]
    levels = [configs.build_level(d, device=local) for d in defs]
    spans = [shard.shard_range(n, rank, world) for n in counts_total]
    first = [f for f, _ in spans]
    counts = [c for _, c in spans]
    upd = [lv.info["dof_updates_per_solve"] for lv in levels]
    per_pair = [upd[l] + (upd[l - 1] if l else 0.0) for l in range(len(levels))]
    total_updates = sum(n * per_pair[l] for l, n in enumerate(counts_total))

    dev = torch.device("cuda", local)
    d_dq = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in counts]
    d_qf = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in counts]
    d_mom = torch.zeros(4 * len(levels), dtype=torch.float64, device=dev)
    streams = [torch.cuda.ExternalStream(lv.stream, device=dev) for lv in levels]
    main = torch.cuda.current_stream(dev)

    def step_device(sequential=False):
        d_mom.zero_()
        ev0 = torch.cuda.Event()
        ev0.record(main)
        for l, lv in enumerate(levels):
            if counts[l] == 0:
                continue
            streams[l].wait_event(ev0)
            wavemc.eval_pairs_device(lv, levels[l - 1] if l else None, 0, l, first[l], counts[l],
                                     d_dq[l].data_ptr(), d_qf[l].data_ptr())
            wavemc.moments_device(lv, d_dq[l].data_ptr(), d_qf[l].data_ptr(), counts[l],
                                  d_mom.data_ptr() + 8 * 4 * l)
            if sequential:  # profiling: kernels of one level at a time
                wavemc.synchronize(lv)
        for l in range(len(levels)):
            e = torch.cuda.Event()
            e.record(streams[l])
            main.wait_event(e)
        if dist is not None:
            dist.all_reduce(d_mom)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize(dev)

    # warm-up, then K timed steps bracketed by barrier + synchronize
    for _ in range(args.warmup):
        step_device()
    barrier()
    launches0 = wavemc.launch_count()
    with ClockSampler(local) as clocks:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(main)
        for _ in range(args.steps):
            step_device()
        end.record(main)
        barrier()
    launches = wavemc.launch_count() - launches0
    ms = start.elapsed_time(end) / args.steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_updates / (ms * 1e-3)
    mom = d_mom.cpu().tolist()

    # e2e: the public host API (per-sample results D2H + host fold in index
    # order) per step, plus the allreduce of the per-level sums
    def step_e2e():
        stats = wavemc.run_mlmc_fixed(levels, counts, 0, first)
        return shard.allreduce_level_sums(stats, device=dev)

    step_e2e()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, min(args.steps, 2))
    t0.record(main)
    for _ in range(e2e_steps):
        stats = step_e2e()
    t1.record(main)
    barrier()
    e2e_ms = t0.elapsed_time(t1) / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    d2h = sum(16 * c + 4 * c * (2 if l else 1) for l, c in enumerate(counts))

    # MLMC time-to-RMSE: the adaptive driver (reference run_mlmc, batched)
    # from scratch to convergence at TTR_EPS, wall time around the public call
    ttr = None
    if world == 1 and args.config == 1:
        costs = [lv.info["dof_updates_per_solve"] for lv in levels]
        wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=TTR_EPS * 4))  # warm-up
        torch.cuda.synchronize(dev)
        runs = []
        for _ in range(3):  # the median of three runs from scratch (each ~0.1 s, host-jitter sensitive)
            t_0 = time.perf_counter()
            res = wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=TTR_EPS))
            runs.append(time.perf_counter() - t_0)
        ttr = {"eps": TTR_EPS, "seconds": sorted(runs)[1], "runs_s": runs, "rmse": res.rmse,
               "converged": res.converged, "estimate": res.estimate, "N_l": [lv["n_samples"] for lv in res.levels]}

    # kernel-level profile pass (not timed above): per-kernel device time
    roofline, kernels = None, None
    if not args.no_profile:
        for lv in levels:
            wavemc.profile_enable(lv, True)
        step_device(sequential=True)
        torch.cuda.synchronize(dev)
        prof = []
        for lv in levels:
            prof.append(wavemc.profile_read(lv))
            wavemc.profile_enable(lv, False)
        roofline, kernels = roofline_from_profile(levels, counts, prof, ms)

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    if roofline is not None:
        peak = peaks.get("hbm_gbs", 6650.0)
        roofline["peak"] = peak
        roofline["frac"] = roofline["achieved"] / peak
        roofline["peak_source"] = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback"

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-based RNG draws, seed 0)",
            "config": {"workload": label,
                       "N_l": counts_total, "levels": [{"n": lv.info["n"], "n_r": lv.info["n_r"], "p": lv.info["p"],
                                                        "n_steps": lv.info["n_steps"]} for lv in levels],
                       "dof_updates_per_step": total_updates, "parallelism": f"samples sharded over {world} GPU(s)",
                       "l2": "inputs (state 2 x n x batch x 8 B per level) exceed L2 at levels 2-4; no flush"},
            "e2e": {"value": total_updates / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": launches, "clocks": clocks.summary(),
            "moments": [{"level": l, "sum_dq": mom[4 * l], "sum_dq2": mom[4 * l + 1], "sum_q": mom[4 * l + 2],
                         "sum_q2": mom[4 * l + 3]} for l in range(len(levels))],
            "variance": [s["variance"] for s in stats]}
    if ttr is not None:
        line["time_to_rmse"] = ttr
    if roofline is not None:
        line["roofline"] = roofline
        line["kernels"] = kernels
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        try:
            cb = cpu_baseline(defs, threads, cpu_T)
            line["cpu_baseline"] = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
                                    "sample": f"config {args.config} bounded sample N_l={cb['counts']}"
                                              + (f", T={cpu_T!r}" if cpu_T is not None else "")
                                              + f", {cb['seconds']:.1f} s"
                                              + (f"; {cb['note']}" if cb.get("note") else "")}
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": f"failed: {exc}"}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def roofline_from_profile(levels, counts, prof, step_ms):
    """Per-kernel device time from the profiled pass, and the roofline of the
    dominant HBM-bound kernel.  Algorithmic bytes per launch (per sample):
      sweep                  8 B x (n reads of z_n + (n - |R|) reads of z_{n-1}
                             + n writes of z_{n+1} or g)
      on-chip substep        8 B x 2 |R| (g in, d_p out) -- on-chip bound
      HBM-resident substep   8 B x 4 |R| per substep (d_m, d_{m-1}, g in,
                             d_{m+1} out) + 8 B x 2 |R| on the last (z_n, z_{n-1})
      R update               8 B x 4 |R|"""
    fused_lv = [bool(lv.info.get("fused")) for lv in levels]
    sweep_ms = sum(p["sweep_ms"] for p in prof)
    sub_ms = sum(p["sub_ms"] for p, f in zip(prof, fused_lv) if not f)
    fused_ms = sum(p["sub_ms"] for p, f in zip(prof, fused_lv) if f)
    upd_ms = sum(p["upd_ms"] for p in prof)
    sweep_bytes = sub_bytes = sub_flops = sub_updates = 0.0
    fused_bytes = fused_updates = fused_flops = 0.0
    global_path = any(lv.info["substep_path"] in (3, 4) for lv in levels)
    for l, lv in enumerate(levels):
        for lvl in ([l] + ([l - 1] if l else [])):
            info = levels[lvl].info
            n, nr, steps, p = info["n"], info["n_r"], info["n_steps"], info["p"]
            c = counts[l]
            if fused_lv[lvl]:
                # whole solves on chip: HBM sees z_0 and the QoI only; the
                # SURVEY 8(d) algorithmic figure (24 B per DOF per global step)
                # is reported as the HBM-equivalent rate of the same work
                fused_bytes += 24.0 * c * steps * n
                fused_updates += c * info["dof_updates_per_solve"]
                fused_flops += c * (steps - 1) * ((p - 1) * (2.0 * info["ap_nnz"] + 7.0 * nr) + 2.0 * info["nnz"])
                continue
            sweep_bytes += 8.0 * c * (steps - 1) * (2 * n + (n - nr))
            if info["substep_path"] == 4:
                # nested tiers: p^k stages of tier k per step, each reading
                # r_k, E_m, E_{m-1} and writing E_{m+1} (or r_k+1) on R_k,
                # plus z_n, z_{n-1} in and z_{n+1} out on R_1
                pk, b, u = 1, 3.0 * nr, 0.0
                for k, nrk in enumerate(info["n_r_tier"]):
                    pk *= p
                    b += 4.0 * pk * nrk
                    u += (pk - pk // p) * nrk
                sub_bytes += 8.0 * c * (steps - 1) * b
                sub_updates += c * (steps - 1) * u
                continue
            if info["substep_path"] == 3:
                sub_bytes += 8.0 * c * (steps - 1) * (4 * nr * (p - 1) + 2 * nr)
            elif info["substep_path"] in (1, 2):
                sub_bytes += 8.0 * c * (steps - 1) * 2 * nr
            sub_flops += c * (steps - 1) * (p - 1) * (2.0 * info["ap_nnz"] + 7.0 * nr)
            sub_updates += c * (steps - 1) * (p - 1) * nr
    gbps = lambda b, ms: b / (ms * 1e-3) / 1e9 if ms else None  # noqa: E731
    kernels = {"sweep": {"ms": sweep_ms, "launches": sum(p["sweep_launches"] for p in prof),
                         "share_of_step": sweep_ms / step_ms if step_ms else None,
                         "achieved_GBps": gbps(sweep_bytes, sweep_ms)},
               "substep": {"ms": sub_ms, "launches": sum(p["sub_launches"] for p in prof),
                           "path": ("hbm-resident nested tiers" if any(lv.info["substep_path"] == 4 for lv in levels)
                                    else ("on-chip + hbm-resident" if any(lv.info["substep_path"] in (1, 2) and not f
                                                                          for lv, f in zip(levels, fused_lv))
                                          else "hbm-resident") if global_path else "on-chip"),
                           "share_of_step": sub_ms / step_ms if step_ms else None,
                           "fp64_TFLOPs": sub_flops / (sub_ms * 1e-3) / 1e12 if sub_ms and sub_flops else None,
                           "substep_dof_updates_per_s": sub_updates / (sub_ms * 1e-3) if sub_ms else None,
                           "achieved_GBps": gbps(sub_bytes, sub_ms)},
               "r_update": {"ms": upd_ms, "launches": sum(p["upd_launches"] for p in prof),
                            "share_of_step": upd_ms / step_ms if step_ms else None}}
    if fused_ms:
        kernels["fused_solve"] = {
            "ms": fused_ms, "levels": [i for i, f in enumerate(fused_lv) if f],
            "launches": sum(p["sub_launches"] for p, f in zip(prof, fused_lv) if f),
            "share_of_step": fused_ms / step_ms if step_ms else None,
            "bound": "on-chip (shared-memory wavefronts + latency; no per-step HBM traffic)",
            "dof_updates_per_s": fused_updates / (fused_ms * 1e-3),
            "fp64_TFLOPs": fused_flops / (fused_ms * 1e-3) / 1e12,
            "hbm_equivalent_GBps": gbps(fused_bytes, fused_ms),
            "note": "HBM-equivalent = SURVEY 8(d) algorithmic 24 B per DOF per global step over the kernel time"}
    # DRAM traffic per launch: the measured/algorithmic ratio of the committed
    # ncu capture (profiles/traffic.json) times this run's algorithmic bytes
    # per launch
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            cap = json.load(f)
    except OSError:
        cap = {}

    def traffic(key, alg_bytes, launches):
        c = cap.get(key) or {}
        if not launches or not c.get("algorithmic_bytes"):
            return None, None
        return c["dram_bytes"] / c["algorithmic_bytes"] * alg_bytes / launches, c.get("launch")

    if global_path and sub_ms >= sweep_ms:
        tiers = any(lv.info["substep_path"] == 4 for lv in levels)
        key = "tier_stage" if tiers else "global_substep"
        t, src = traffic(key, sub_bytes, kernels["substep"]["launches"])
        roof = {"bound": "hbm", "kernel": key, "achieved": kernels["substep"]["achieved_GBps"],
                "unit": "GB/s", "traffic": t, "traffic_capture": src,
                "note": ("dominant kernel, HBM-resident substeps (algorithmic bytes); traffic per global step's "
                         "group of substep launches")}
    elif not sweep_ms and fused_ms:
        # every level runs the fused on-chip solve (e.g. config 0): no HBM
        # stream per step; report its SURVEY 8(d) HBM-equivalent rate
        roof = {"bound": "hbm", "kernel": "fused_solve", "achieved": kernels["fused_solve"]["hbm_equivalent_GBps"],
                "unit": "GB/s", "traffic": None, "traffic_capture": None,
                "note": ("HBM-equivalent rate of the fused lattice solve (24 B per DOF per global step over its "
                         "time); the state never leaves the SM, the kernel is bound on chip "
                         "(kernels.fused_solve), so this fraction is not its limiter")}
    else:
        t, src = traffic("sweep", sweep_bytes, kernels["sweep"]["launches"])
        roof = {"bound": "hbm", "kernel": "sweep", "achieved": kernels["sweep"]["achieved_GBps"], "unit": "GB/s",
                "traffic": t, "traffic_capture": src,
                "note": ("HBM roofline of the sweep kernel (algorithmic bytes, levels without the fused solve); "
                         "the dominant kernels keep the state on chip and are shared-memory bound, see "
                         "kernels.fused_solve / kernels.substep")}
    return roof, kernels


def kl_table_file(tmp):
    from paper_2106_11117_b200 import configs, wavemc
    kl = configs.KL_FIELD
    table, _ = wavemc.kl_table(kl["cells"][0], kl["cells"][1], kl["sigma"], kl["corr_len"], kl["modes"])
    path = os.path.join(tmp, "kl.txt")
    with open(path, "w") as f:
        f.write(f"{table.shape[0]} {table.shape[1]}\n")
        f.write("\n".join(repr(float(v)) for v in table.ravel()) + "\n")
    return path, {"kl-table": path, "cells-x": kl["cells"][0], "cells-y": kl["cells"][1]}


def adaptive_arm(args, world, rank, local):
    """Config 4: one step = the adaptive MLMC estimator (reference run_mlmc
    algorithm) from scratch to the RMSE target; metric DOF-updates/s of the
    work it performed, plus the time-to-RMSE itself."""
    from paper_2106_11117_b200 import configs
    eps = args.eps or configs.CONFIG4_EPS
    defs = configs.config4()
    if args.impl == "reference":
        if rank != 0:
            return 0
        import oracle_py
        threads = os.cpu_count() or 1
        tmp = tempfile.mkdtemp(prefix="wmc_c4_")
        _, klargs = kl_table_file(tmp)
        specs = []
        for l, d in enumerate(defs):
            p = os.path.join(tmp, f"l{l}.mesh")
            configs.build_mesh(d).dump(p)
            specs.append((p, d.dt, d.substeps))
        runs = [oracle_py.RefDriver().adaptive(specs, eps, threads=threads, **klargs)
                for _ in range(args.warmup + args.steps)][args.warmup:]
        shutil.rmtree(tmp, ignore_errors=True)
        sec = sum(r["seconds"] for r in runs) / len(runs)
        line = {"impl": "reference", "metric": "MLMC time-to-RMSE", "value": sec, "unit": "s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (counter-based RNG, Box-Muller KL weights, seed 0)",
                "config": {"workload": f"BASELINE config 4: adaptive MLMC to RMSE {eps}, log-normal KL", "eps": eps},
                "cpu_baseline": {"value": sec, "unit": "s", "cores": threads, "kind": "reference",
                                 "sample": f"full adaptive run, reference run_mlmc, {threads} threads"},
                "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "N_l": [lv["N"] for lv in runs[0]["levels"]], "estimate": runs[0]["estimate"]}
        print(json.dumps(line))
        return 0
    import torch
    from paper_2106_11117_b200 import wavemc
    torch.cuda.set_device(local)
    levels = [configs.build_level(d, device=local, kl=True) for d in defs]
    costs = [lv.info["dof_updates_per_solve"] for lv in levels]
    for _ in range(args.warmup):
        wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=eps))
    torch.cuda.synchronize()
    launches0 = wavemc.launch_count()
    times, res = [], None
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            res = wavemc.run_mlmc(levels, costs, wavemc.MlmcConfig(eps=eps))
            times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    work = sum(lv["cost"]["dof_updates"] for lv in res.levels)
    line = {"metric": "MLMC time-to-RMSE", "value": sec, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-based RNG, Box-Muller KL weights, seed 0)",
            "config": {"workload": f"BASELINE config 4: adaptive MLMC to RMSE {eps}, log-normal KL (sigma 0.5, "
                                   "l 0.1, 64 modes, 16x16 cells), config-1 geometry", "eps": eps},
            "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 16 * sum(lv["n_samples"] for lv in res.levels)},
            "gpu_launches": (wavemc.launch_count() - launches0) // max(1, args.steps), "clocks": clocks.summary(),
            "dof_updates_per_s": work / sec, "rmse": res.rmse, "converged": res.converged,
            "estimate": res.estimate, "N_l": [lv["n_samples"] for lv in res.levels]}
    if rank == 0:
        print(json.dumps(line))
    return 0


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.config == 4:
        return adaptive_arm(args, world, rank, local)
    if args.impl == "reference":
        return reference_arm(args, world, rank)
    return b200_arm(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
