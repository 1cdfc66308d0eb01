"""Summarise ncu captures (gpurun_out/) into markdown for profiles/.

  python tools/summarize_profiles.py launches gpurun_out/launches.csv
  python tools/summarize_profiles.py report gpurun_out/prof_lattice.ncu-rep
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Block Size", "Grid Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__sass_thread_inst_executed_op_dfma_pred_on.sum"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0].split("::")[-1]
        tot[name] += float(r[idx["Metric Value"]].replace(",", ""))
        cnt[name] += 1
    total = sum(tot.values())
    print("| kernel | launches | total (us) | share | mean (us) |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {100 * v / total:.1f} % | {v / cnt[k] / 1e3:.2f} |")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    seen = {}
    name = ""
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get("ID") != "0":
            continue
        name = d.get("Kernel Name", name)
        if d["Metric Name"] in KEYS and d["Metric Name"] not in seen:
            seen[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh, ru, rv = rr[0], rr[1], rr[2]
    print(f"kernel: `{name[:110]}`\n")
    print("| metric | value |")
    print("|---|---|")
    for k in KEYS:
        if k in seen:
            print(f"| {k} | {seen[k]} |")
    for h, u, v in zip(rh, ru, rv):
        if h in RAW:
            print(f"| `{h}` | {v} {u} |")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
