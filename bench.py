#!/usr/bin/env python
"""Benchmark of the batched LF-LTS MLMC hot path (BASELINE.json config 1).

One step = the whole fixed-N MLMC estimator of config 1: coupled pairs on
levels 0..4 (h_l = 1/16..1/256, p_l = 32..2, N_l = 65536, 16384, 4096, 1024,
256), both solves of every pair, FP64, plus the per-level moment sums and
(N > 1) one NCCL allreduce of them.  Metric: DOF-updates/s with
U = n + (p-1)|R| per global step per solve.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 0..4] [--integrator lts|lf]

--gpus N > 1 re-launches itself under torch.distributed.run (N ranks, one
per GPU, NCCL).  Rank r evaluates whole 64-sample granules of every level
(balanced over the levels, shard.shard_levels) with streams keyed by the
global index, so per-sample results do not depend on N; total work is fixed
("strong" scaling).
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
# the paper's per-sample model cost ratio C_l^LF / C_l^LTS of its 2D channel
# (PAPER.md:1067-1070), context for the measured LTS/LF time ratios
PAPER_LF_OVER_LTS = [5.89, 7.82, 4.54, 2.51]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--scale", type=float, default=None,
                    help="fraction of N_l (default 1.0 = the BASELINE counts; config 3: 1/32, one whole "
                         "256-sample batch of the 8192 -- the full set is 32 such batches, ~10 min per step)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4],
                    help="BASELINE config: 1 (default, MLMC), 0 (single-level MC), 2 (graded L-shape MLMC, "
                         "nested 3-tier LTS), 3 (large single level), 4 (adaptive MLMC to an RMSE target, "
                         "log-normal KL coefficient)")
    ap.add_argument("--integrator", default="lts", choices=["lts", "lf"],
                    help="config 1: lf = the global leap-frog comparison arm (dt = 0.2 h_min on every level); "
                         "the line then carries the measured LF / LTS time ratios")
    ap.add_argument("--eps", type=float, default=None, help="config 4: RMSE target (default BASELINE 1e-3)")
    ap.add_argument("--field", default="cells", choices=["cells", "element"],
                    help="config 4: KL field on the 32 x 32 cell grid, or at every triangle's centroid")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(args) -> int:
    """--gpus N without a launcher: re-run this script under
    torch.distributed.run, N ranks on this node, rendezvous on 127.0.0.1."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "cores": os.cpu_count() or 1}


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return {}


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
# workloads

def workload(config: int, integrator: str = "lts"):
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
    if integrator == "lf":
        return configs.config1("lf"), list(configs.CONFIG1_COUNTS), (
            "BASELINE config 1, global leap-frog arm: fixed-N MLMC, 5 levels h=1/16..1/256, dt=0.2 h_min"), None
    return configs.config1(), list(configs.CONFIG1_COUNTS), (
        "BASELINE config 1: fixed-N MLMC, LF-LTS, 5 levels h=1/16..1/256, p=32..2"), None


# ---------------------------------------------------------------------------
# CPU baselines: the reference compiled from its own sources (oracle/_ref),
# else our C restatement.  Inputs (meshes, level data) come from a separate
# process (tools/dump_inputs.py) so the timed reference arm never maps the
# product library.

def dump_inputs(config: int, final_time=None, lf=False, kl=False, kl_element=False) -> dict:
    tmp = tempfile.mkdtemp(prefix="wmc_inputs_")
    cmd = [sys.executable, os.path.join(ROOT, "tools", "dump_inputs.py"), "--config", str(config), "--out", tmp]
    if final_time is not None:
        cmd += ["--final-time", repr(final_time)]
    if lf:
        cmd.append("--lf")
    if kl:
        cmd.append("--kl")
    if kl_element:
        cmd.append("--kl-element")
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    inp = load_json(os.path.join(tmp, "inputs.json"))
    inp["dir"] = tmp
    return inp


def ref_sample_counts(threads: int, config: int):
    """Bounded sample for the CPU, in the proportions of N_l, sized for
    ~10-20 s of wall time on `threads` cores."""
    t = max(1, threads)
    if config == 2:  # N_l halving, horizon T/8
        return [8 * t, 4 * t, 2 * t, t, max(1, t // 2)]
    if config in (1, 4):
        return [64 * t, 16 * t, 4 * t, t, max(1, t // 4)]
    return None


def config2_extra(final_time):
    from paper_2106_11117_b200 import configs  # constants only (no library)
    c = configs.CONFIG2_PROBLEM
    return {"T": repr(final_time), "cells-x": c["cells"][0], "cells-y": c["cells"][1], "ic": ",".join(map(repr, c["ic"])),
            "box": ",".join(map(repr, c["qoi_box"])), "domain": ",".join(map(repr, c["domain"])), "qoi-mean": 1}


def run_reference_cpu(config: int, threads: int, final_time=None, lf=False, counts=None):
    """A bounded sample through the unmodified reference library (its own
    sample_delta_q over a run_jobs-style pool of `threads` workers)."""
    import oracle_py
    inp = dump_inputs(config, final_time, lf)
    levels = inp["levels"]
    counts = counts or ref_sample_counts(threads, config) or [4 * threads if final_time is None else threads]
    nested = any(lv["tiers"] > 1 for lv in levels)
    # config 2: the reference has no nested tiers; its own LF-LTS on the same
    # mesh takes P = P_1 and p = 2^tiers (stable at the finest tier)
    specs = [(lv["mesh"], lv["dt"], lv["p"] ** lv["tiers"] if nested else lv["p"]) for lv in levels]
    extra = {"T": repr(final_time)} if final_time is not None else {}
    if nested:
        extra = config2_extra(final_time if final_time is not None else 2.0)
    res = oracle_py.RefDriver().mlmc(specs, counts, kind="lf" if lf else "lts", threads=threads, **extra)
    shutil.rmtree(inp["dir"], ignore_errors=True)
    work = res["dof_updates"]
    if nested:  # the same samples counted in the config-2 (nested) units
        upd = [lv["dof_updates_per_solve"] for lv in levels]
        work = sum(n * (upd[l] + (upd[l - 1] if l else 0.0)) for l, n in enumerate(counts))
    return {"value": work / res["seconds"], "seconds": res["seconds"], "dof_updates": work, "counts": counts,
            "kind": "reference", "cores": res["threads"], "levels": res["levels"],
            "note": ("reference single-tier LF-LTS (P = P_1, p = 8) on the config-2 meshes and samples (it has no "
                     "nested tiers); value = nested-scheme DOF-updates of the same samples / reference time"
                     if nested else None)}


def run_port_cpu(config: int, threads: int, final_time=None):
    """Fallback when oracle/_ref is absent: our C restatement, `threads` workers."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle_py
    from paper_2106_11117_b200 import configs, wavemc
    oracle_py.build()
    orc = oracle_py.COracle()
    defs = workload(config)[0]
    counts = ref_sample_counts(threads, config) or [4 * threads if final_time is None else threads]
    meshes = [oracle_py.MeshArrays(*configs.build_mesh(d).arrays()) for d in defs]
    T = [final_time if final_time is not None else d.final_time for d in defs]
    probs = []
    upd = []
    for d, t in zip(defs, T):
        if d.shape == "lshape":
            c = configs.CONFIG2_PROBLEM
            probs.append(oracle_py.problem(d.dt, d.substeps, final_time=t, cells=c["cells"], ic=c["ic"],
                                           box=c["qoi_box"], domain=c["domain"], qoi_mean=True, tiers=d.tiers))
        else:
            probs.append(oracle_py.problem(d.dt, d.substeps, final_time=t))
        spec = configs.level_spec(d)
        spec.final_time = t
        upd.append(wavemc.level_plan(configs.build_mesh(d), spec)["dof_updates_per_solve"])
    jobs = [(l, i) for l in range(len(defs)) for i in range(counts[l])]

    def one(job):
        l, i = job
        orc.eval_pairs(meshes[l], probs[l], meshes[l - 1] if l else None, probs[l - 1] if l else None, 0, l, i, 1)
        return upd[l] + (upd[l - 1] if l else 0.0)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        total = sum(ex.map(one, jobs))
    dt = time.perf_counter() - t0
    return {"value": total / dt, "seconds": dt, "dof_updates": total, "counts": counts, "kind": "port",
            "cores": threads}


def cpu_baseline(config: int, threads: int, final_time=None, lf=False):
    import oracle_py
    if os.path.exists(oracle_py.REF_DRIVER):
        return run_reference_cpu(config, threads, final_time, lf)
    return run_port_cpu(config, threads, final_time)


def reference_time_to_rmse(threads: int):
    """The reference's own run_mlmc (src/mlmc.cpp:165-233) to RMSE TTR_EPS on
    the config-1 hierarchy, wall time measured by the driver."""
    import oracle_py
    inp = dump_inputs(1)
    specs = [(lv["mesh"], lv["dt"], lv["p"]) for lv in inp["levels"]]
    res = oracle_py.RefDriver().adaptive(specs, TTR_EPS, threads=threads)
    shutil.rmtree(inp["dir"], ignore_errors=True)
    return {"eps": TTR_EPS, "seconds": res["seconds"], "rmse": math.sqrt(res["total_variance"] + res["bias"]),
            "converged": res["converged"], "estimate": res["estimate"], "N_l": [lv["N"] for lv in res["levels"]],
            "threads": res["threads"]}


def reference_lf_over_lts(threads: int):
    """The reference's per-solve time ratio LF / LTS on every config-1 level
    (leapfrog_step at dt = 0.2 h_min against lts_step at dt = 0.2 h_l), from
    a bounded sample of single-level solves timed by its own driver."""
    import oracle_py
    drv = oracle_py.RefDriver()
    out = []
    lts, lf = dump_inputs(1), dump_inputs(1, lf=True)
    try:
        for l, (a, b) in enumerate(zip(lts["levels"], lf["levels"])):
            n = max(1, threads)
            ha, _ = drv.solve(a["mesh"], a["dt"], a["p"], "lts", 0, 0, n, threads=threads)
            hb, _ = drv.solve(b["mesh"], b["dt"], 1, "lf", 0, 0, n, threads=threads)
            out.append(float(hb["seconds"]) / float(ha["seconds"]))
    finally:
        shutil.rmtree(lts["dir"], ignore_errors=True)
        shutil.rmtree(lf["dir"], ignore_errors=True)
    return out


# ---------------------------------------------------------------------------

def reference_arm(args, world, rank):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    _, counts_total, label, cpu_T = workload(args.config, args.integrator)
    lf = args.integrator == "lf"
    try:
        runs = [cpu_baseline(args.config, threads, cpu_T, lf) for _ in range(args.warmup + args.steps)]
    except Exception as exc:  # the oracle always exists; report loudly
        print(json.dumps({"impl": "reference", "unavailable": f"reference CPU run failed: {exc}"}))
        return 0
    timed = runs[args.warmup:]
    value = sum(r["dof_updates"] for r in timed) / sum(r["seconds"] for r in timed)
    ttr = None
    if args.config == 1 and not lf:
        try:
            ttr = reference_time_to_rmse(threads)
        except Exception as exc:
            ttr = {"eps": TTR_EPS, "error": str(exc)}
    r0 = timed[0]
    ci = cpu_info()
    sample = (f"config {args.config} bounded sample N_l={r0['counts']} (of {counts_total}) per step"
              + (f", horizon shortened to T={cpu_T!r}" if cpu_T is not None else "")
              + f", {r0['cores']} threads, {r0['kind']}, {ci['cpu_model']}"
              + (f"; {r0['note']}" if r0.get("note") else ""))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(r["seconds"] for r in timed) / len(timed),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (counter-based RNG draws, seed 0)",
            "config": {"workload": label + " (bounded CPU sample)",
                       "parallelism": f"{r0['cores']} CPU threads ({ci['cpu_model']})"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r0["cores"], "kind": r0["kind"],
                             "cpu_model": ci["cpu_model"], "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "time_to_rmse": ttr}
    print(json.dumps(line))
    return 0


def b200_arm(args, world, rank, local):
    import torch

    from paper_2106_11117_b200 import configs, shard, wavemc

    # more ranks than devices (checking the rank path on a one-GPU box): ranks
    # share devices and the collectives go over gloo on host copies; the line
    # says so ("ranks_share_devices") -- not a scaling measurement
    ndev = max(1, torch.cuda.device_count())
    shared = world > ndev
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allreduce(t, op=None):
        if dist is None:
            return t
        kw = {} if op is None else {"op": op}
        if shared:
            h = t.cpu()
            dist.all_reduce(h, **kw)
            t.copy_(h)
        else:
            dist.all_reduce(t, **kw)
        return t
    lf = args.integrator == "lf"
    defs, counts_total, label, cpu_T = workload(args.config, args.integrator)
    if args.scale is None:
        args.scale = 0.03125 if args.config == 3 else 1.0
    if args.scale != 1.0:
        label += f" (N_l scaled by {args.scale})"
    counts_total = [max(1, int(round(n * args.scale))) for n in counts_total]
    levels = [configs.build_level(d, device=local) for d in defs]
    upd = [lv.info["dof_updates_per_solve"] for lv in levels]
    per_pair = [upd[l] + (upd[l - 1] if l else 0.0) for l in range(len(levels))]
    spans = shard.shard_levels(counts_total, per_pair, world)[rank]
    first = [f for f, _ in spans]
    counts = [c for _, c in spans]
    total_updates = sum(n * per_pair[l] for l, n in enumerate(counts_total))

    dev = torch.device("cuda", local)
    d_dq = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in counts]
    d_qf = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in counts]
    d_mom = torch.zeros(4 * len(levels), dtype=torch.float64, device=dev)
    streams = [torch.cuda.ExternalStream(lv.stream, device=dev) for lv in levels]
    main = torch.cuda.current_stream(dev)

    def step_device(sequential=False, lvls=None, strs=None):
        lvls = lvls or levels
        strs = strs or streams
        d_mom.zero_()
        ev0 = torch.cuda.Event()
        ev0.record(main)
        for l, lv in enumerate(lvls):
            if counts[l] == 0:
                continue
            strs[l].wait_event(ev0)
            wavemc.eval_pairs_device(lv, lvls[l - 1] if l else None, 0, l, first[l], counts[l],
                                     d_dq[l].data_ptr(), d_qf[l].data_ptr())
            wavemc.moments_device(lv, d_dq[l].data_ptr(), d_qf[l].data_ptr(), counts[l],
                                  d_mom.data_ptr() + 8 * 4 * l)
            if sequential:  # profiling: kernels of one level at a time
                wavemc.synchronize(lv)
        for l in range(len(lvls)):
            e = torch.cuda.Event()
            e.record(strs[l])
            main.wait_event(e)
        if dist is not None:
            allreduce(d_mom)

    def barrier():
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize(dev)

    def check_levels():  # device-resident results: the first unstable sample, if any (check_finite)
        for lv in levels:
            wavemc.synchronize(lv)

    # warm-up, then K timed steps bracketed by barrier + synchronize
    for _ in range(args.warmup):
        step_device()
    barrier()
    check_levels()
    launches0 = wavemc.launch_count()
    with ClockSampler(local) as clocks:
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(main)
        for _ in range(args.steps):
            step_device()
        end.record(main)
        barrier()
    check_levels()
    launches = wavemc.launch_count() - launches0
    ms = start.elapsed_time(end) / args.steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        allreduce(t, dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_updates / (ms * 1e-3)
    mom = d_mom.cpu().tolist()

    # e2e: the public host API (per-sample results D2H + host fold in index
    # order) per step, plus the allreduce of the per-level sums; the same K
    # steps as the device timing
    def step_e2e():
        stats = wavemc.run_mlmc_fixed(levels, counts, 0, first)
        return shard.allreduce_level_sums(stats, device=None if shared else dev)

    step_e2e()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    for _ in range(args.steps):
        stats = step_e2e()
    t1.record(main)
    barrier()
    e2e_ms = t0.elapsed_time(t1) / args.steps
    if dist is not None:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        allreduce(t, dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    d2h = sum(16 * c + 4 * c * (2 if l else 1) for l, c in enumerate(counts))

    # MLMC time-to-RMSE: the adaptive driver (reference run_mlmc, batched)
    # from scratch to convergence at TTR_EPS, wall time around the public call
    ttr = None
    if world == 1 and args.config == 1 and not lf:
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

    # config-1 global leap-frog arm: the LTS estimator timed in the same run
    # and the per-level LF / LTS solve-time ratios (device and reference CPU)
    lf_vs_lts = None
    if lf and args.config == 1:
        lts_levels = [configs.build_level(d, device=local) for d in configs.config1()]
        lts_streams = [torch.cuda.ExternalStream(lv.stream, device=dev) for lv in lts_levels]
        for _ in range(max(1, args.warmup)):
            step_device(lvls=lts_levels, strs=lts_streams)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for _ in range(args.steps):
            step_device(lvls=lts_levels, strs=lts_streams)
        b.record(main)
        barrier()
        lts_ms = a.elapsed_time(b) / args.steps
        per_level = []
        for l in range(len(levels)):  # one 1024-sample batch of single solves per level and integrator
            ts = []
            for lv in (levels[l], lts_levels[l]):
                n = 1024
                buf = torch.empty(n, dtype=torch.float64, device=dev)
                wavemc.eval_pairs_device(lv, None, 0, l, 0, n, buf.data_ptr(), buf.data_ptr())
                wavemc.synchronize(lv)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s = torch.cuda.ExternalStream(lv.stream, device=dev)
                e0.record(s)
                wavemc.eval_pairs_device(lv, None, 0, l, 0, n, buf.data_ptr(), buf.data_ptr())
                e1.record(s)
                wavemc.synchronize(lv)
                ts.append(e0.elapsed_time(e1))
            per_level.append(ts[0] / ts[1])
        lf_vs_lts = {"estimator_time_ratio_lf_over_lts": ms / lts_ms, "lts_estimator_ms": lts_ms,
                     "per_level_solve_time_ratio_lf_over_lts": per_level,
                     "paper_model_cost_ratio_lf_over_lts_channel2d": PAPER_LF_OVER_LTS,
                     "note": "per-level ratios: one batch of 1024 single solves per integrator on the device"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            try:
                lf_vs_lts["reference_cpu_per_level_solve_time_ratio_lf_over_lts"] = reference_lf_over_lts(
                    os.cpu_count() or 1)
            except Exception as exc:
                lf_vs_lts["reference_cpu_error"] = str(exc)

    # kernel-level profile pass (not timed above): per-kernel device time
    roofline, kernels, step_frac = None, None, None
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    fp64 = load_json(os.path.join(ROOT, "profiles", "fp64_peak.json"))
    if not args.no_profile:
        for lv in levels:
            wavemc.profile_enable(lv, True)
        step_device(sequential=True)
        torch.cuda.synchronize(dev)
        prof = []
        for lv in levels:
            prof.append(wavemc.profile_read(lv))
            wavemc.profile_enable(lv, False)
        roofline, kernels, step_bytes = roofline_from_profile(levels, counts, prof, ms, peaks, fp64)
        step_frac = {"bytes_per_step": step_bytes, "achieved_GBps": step_bytes / (ms * 1e-3) / 1e9,
                     "peak_GBps": peaks.get("hbm_gbs", 6650.0),
                     "frac": step_bytes / (ms * 1e-3) / 1e9 / peaks.get("hbm_gbs", 6650.0),
                     "note": "SURVEY 8(d) algorithmic bytes (24 B per DOF per solve per global step) of the whole "
                             "step over ms_per_step, against the measured HBM copy peak"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (counter-based RNG draws, seed 0)",
            "config": {"workload": label,
                       "N_l": counts_total, "levels": [{"n": lv.info["n"], "n_r": lv.info["n_r"], "p": lv.info["p"],
                                                        "n_steps": lv.info["n_steps"],
                                                        "path": lv.info["substep_path"]} for lv in levels],
                       "dof_updates_per_step": total_updates,
                       "parallelism": f"samples sharded over {world} GPU(s) in 64-sample granules",
                       "l2": "inputs (state 2 x n x batch x 8 B per level) exceed L2 at levels 2-4; no flush"},
            "e2e": {"value": total_updates / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": args.steps,
                    "note": "inputs are seeds (per-sample coefficients drawn on the device); per-sample dQ, Q and "
                            "fail flags copied D2H and folded on the host every step"},
            "gpu_launches": launches, "clocks": clocks.summary(),
            "ranks_share_devices": shared,
            "moments": [{"level": l, "sum_dq": mom[4 * l], "sum_dq2": mom[4 * l + 1], "sum_q": mom[4 * l + 2],
                         "sum_q2": mom[4 * l + 3]} for l in range(len(levels))],
            "variance": [s["variance"] for s in stats]}
    if ttr is not None:
        line["time_to_rmse"] = ttr
    if lf_vs_lts is not None:
        line["lf_vs_lts"] = lf_vs_lts
    if roofline is not None:
        line["roofline"] = roofline
        line["step_frac"] = step_frac
        line["kernels"] = kernels
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        ci = cpu_info()
        try:
            cb = cpu_baseline(args.config, threads, cpu_T, lf)
            line["cpu_baseline"] = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"],
                                    "cpu_model": ci["cpu_model"],
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


def roofline_from_profile(levels, counts, prof, step_ms, peaks, fp64):
    """Per-kernel-class device time from the profiled pass (CUDA events on
    the level streams), the roofline of each class and of the dominant one
    (largest share of the step).  Algorithmic bytes: 24 B per
    DOF per solve per global step, split over the kernels that move them:
      sweep          8 B x (z_n reads + z_{n-1} reads + z_{n+1} / g writes) of its rows
      tiled step     8 B x 3 |R| (z_n, z_{n-1} in, z_{n+1} out of R)
      fused solve    24 B x n (the whole step on chip: its HBM-equivalent rate)
      HBM substeps   8 B x (4 |R| per substep + 2 |R|) (their own bytes, above 8(d))
    FP64 flops (algorithmic): 2 per operator entry of every product plus 7 per
    R row and substep (the recursion)."""
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    fp64_peak = fp64.get("fp64_tflops", 37.08)
    traffic = load_json(os.path.join(ROOT, "profiles", "traffic.json"))
    cls = {}

    def add(name, ms, launches, bytes_=0.0, flops=0.0, updates=0.0, alg8d=0.0, solves=0):
        c = cls.setdefault(name, {"ms": 0.0, "launches": 0, "bytes": 0.0, "flops": 0.0, "updates": 0.0, "alg8d": 0.0,
                                  "solves": 0})
        c["solves"] += solves
        c["ms"] += ms
        c["launches"] += launches
        c["bytes"] += bytes_
        c["flops"] += flops
        c["updates"] += updates
        c["alg8d"] += alg8d

    step_bytes = 0.0
    # a level's profile covers every solve of that level (the fine role of
    # its own pairs and the coarse role of the next level's pairs)
    for lvl, lv in enumerate(levels):
        c = counts[lvl] + (counts[lvl + 1] if lvl + 1 < len(levels) else 0)
        info = lv.info
        n, nr, steps, p = info["n"], info["n_r"], info["n_steps"], info["p"]
        path = info["substep_path"]
        p_ = prof[lvl]
        step_bytes += 24.0 * c * steps * n
        flops = c * (steps - 1) * ((p - 1) * (2.0 * info["ap_nnz"] + 7.0 * nr) + 2.0 * info["nnz"])
        if info.get("fused"):
            add("fused_solve", p_["sub_ms"], p_["sub_launches"], 24.0 * c * steps * n, flops,
                c * info["dof_updates_per_solve"], 24.0 * c * steps * n, solves=c)
            continue
        if path == 5:  # tiled: the sweep covers the rows outside R, the tile kernel R
            sweep_b = 24.0 * c * (steps - 1) * (n - nr)
            sub_b = 24.0 * c * (steps - 1) * nr
        else:
            sweep_b = 8.0 * c * (steps - 1) * (2 * n + (n - nr))
            sub_b = 0.0
            if path == 3:
                sub_b = 8.0 * c * (steps - 1) * (4 * nr * (p - 1) + 2 * nr)
            elif path in (1, 2):
                sub_b = 8.0 * c * (steps - 1) * 2 * nr
        sub_u = c * (steps - 1) * (p - 1) * nr
        if p_["sweep_ms"]:
            add("sweep", p_["sweep_ms"], p_["sweep_launches"], sweep_b)
        if path == 5:
            add("tiled_step", p_["sub_ms"], p_["sub_launches"], sub_b, flops, sub_u, sub_b)
        elif path == 3:
            add("global_substep", p_["sub_ms"], p_["sub_launches"], sub_b, flops, sub_u)
        elif path == 4:
            # nested tiers: tier k runs p^(k-1) times per step; stage 0 over the rows
            # outside R_(k+1) (r_k in, E_1 out), stages m >= 1 over all of R_k (r_k and
            # E_m in, E_(m+1) or r_(k+1) out, E_(m-1) in from m = 2); the last stage of
            # tier 1 also reads z_n, z_(n-1) and writes z_(n+1) on R_1
            rk = info["n_r_tier"] + [0]
            tier_b, runs = 3.0 * rk[0], 1
            for k in range(info["tiers"]):
                own = rk[k] - rk[k + 1]
                tier_b += runs * (2.0 * own + (p - 1) * 3.0 * rk[k] + max(0, p - 2) * own)
                runs *= p
            add("tier_stage", p_["sub_ms"], p_["sub_launches"], 8.0 * c * (steps - 1) * tier_b, flops, sub_u)
        elif path in (1, 2):
            add("onchip_substep", p_["sub_ms"], p_["sub_launches"], sub_b, flops, sub_u)
        if p_["upd_ms"]:
            add("r_update", p_["upd_ms"], p_["upd_launches"])
    kernels = {}
    for name, c in cls.items():
        k = {"ms": c["ms"], "launches": c["launches"], "share_of_step": c["ms"] / step_ms if step_ms else None}
        if c["bytes"] and c["ms"]:
            k["achieved_GBps"] = c["bytes"] / (c["ms"] * 1e-3) / 1e9
            k["hbm_frac"] = k["achieved_GBps"] / hbm_peak
        if c["flops"] and c["ms"]:
            k["fp64_TFLOPs"] = c["flops"] / (c["ms"] * 1e-3) / 1e12
            k["fp64_frac"] = k["fp64_TFLOPs"] / fp64_peak
        if c["updates"] and c["ms"]:
            k["dof_updates_per_s"] = c["updates"] / (c["ms"] * 1e-3)
        tr = traffic.get(name) or {}
        if tr.get("dram_bytes_per_solve") and c["launches"] and c.get("solves"):
            k["traffic_per_launch"] = tr["dram_bytes_per_solve"] * c["solves"] / c["launches"]
            k["traffic_capture"] = tr.get("launch")
        elif tr.get("algorithmic_bytes") and c["launches"] and c["bytes"]:
            k["traffic_per_launch"] = tr["dram_bytes"] / tr["algorithmic_bytes"] * c["bytes"] / c["launches"]
            k["traffic_capture"] = tr.get("launch")
        kernels[name] = k
    dom = max(cls, key=lambda q: cls[q]["ms"])
    k = kernels[dom]
    if dom in ("fused_solve", "tiled_step", "onchip_substep"):
        # on-chip kernels: bound by FP64 issue / latency, not HBM; the SURVEY
        # 8(d) HBM-equivalent rate beside it
        roof = {"bound": "fp64", "kernel": dom, "achieved": k.get("fp64_TFLOPs"), "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": k.get("fp64_frac"),
                "peak_source": "measured (profiles/fp64_peak.json, tools/fp64_peak.cu)",
                "hbm_equivalent": {"achieved": cls[dom]["alg8d"] / (cls[dom]["ms"] * 1e-3) / 1e9
                                   if cls[dom]["alg8d"] else k.get("achieved_GBps"),
                                   "peak": hbm_peak, "unit": "GB/s"},
                "traffic": k.get("traffic_per_launch"), "share_of_step": k["share_of_step"]}
        he = roof["hbm_equivalent"]
        he["frac"] = he["achieved"] / hbm_peak if he["achieved"] else None
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": k.get("achieved_GBps"), "peak": hbm_peak, "unit": "GB/s",
                "frac": k.get("hbm_frac"), "traffic": k.get("traffic_per_launch"),
                "share_of_step": k["share_of_step"]}
    roof["peak_hbm_source"] = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    roof["secondary"] = {name: {q: v for q, v in kk.items() if q in ("share_of_step", "achieved_GBps", "hbm_frac",
                                                                     "fp64_TFLOPs", "fp64_frac")}
                         for name, kk in kernels.items() if name != dom}
    return roof, kernels, step_bytes


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
        inp = dump_inputs(4, kl=True, kl_element=args.field == "element")
        specs = [(lv["mesh"], lv["dt"], lv["p"]) for lv in inp["levels"]]
        runs = [oracle_py.RefDriver().adaptive(specs, eps, threads=threads, **inp["kl"])
                for _ in range(args.warmup + args.steps)][args.warmup:]
        shutil.rmtree(inp["dir"], ignore_errors=True)
        sec = sum(r["seconds"] for r in runs) / len(runs)
        ci = cpu_info()
        line = {"impl": "reference", "metric": "MLMC time-to-RMSE", "value": sec, "unit": "s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (counter-based RNG, Box-Muller KL weights, seed 0)",
                "config": {"workload": f"BASELINE config 4: adaptive MLMC to RMSE {eps}, log-normal KL"
                                       + (" at the element centroids" if args.field == "element" else ""), "eps": eps},
                "cpu_baseline": {"value": sec, "unit": "s", "cores": threads, "kind": "reference",
                                 "cpu_model": ci["cpu_model"],
                                 "sample": f"full adaptive run, reference run_mlmc, {threads} threads"},
                "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "N_l": [lv["N"] for lv in runs[0]["levels"]], "estimate": runs[0]["estimate"]}
        print(json.dumps(line))
        return 0
    import torch
    from paper_2106_11117_b200 import wavemc
    torch.cuda.set_device(local)
    levels = [configs.build_level(d, device=local, kl="element" if args.field == "element" else True) for d in defs]
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
                                   "l 0.1, 64 modes, " + ("per element" if args.field == "element" else "32x32 cells")
                                   + "), config-1 geometry", "eps": eps},
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.config == 4:
        return adaptive_arm(args, world, rank, local)
    if args.impl == "reference":
        return reference_arm(args, world, rank)
    return b200_arm(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
