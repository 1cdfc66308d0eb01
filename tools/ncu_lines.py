"""Top CUDA source lines of one kernel by warp-stall samples, from
`ncu -i REP --page source --csv --print-source=cuda,sass` (line aggregates:
rows whose address column is '-')."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if r and r[0] == "Line No")
i_stall = hdr.index("Warp Stall Sampling (All Samples)")
i_inst = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if len(r) > i_stall and r[0].isdigit() and r[2] == "-":
        try:
            lines.append((int(r[i_stall]), int(r[i_inst] or 0), int(r[0]), r[1]))
        except ValueError:
            pass
tot = sum(x[0] for x in lines) or 1
print(f"total stall samples {tot}")
for st, ins, ln, src in sorted(lines, reverse=True)[:n_top]:
    print(f"{100 * st / tot:5.1f}% {ins:>11d}  {ln:5d}  {src.strip()[:90]}")
