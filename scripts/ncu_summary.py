#!/usr/bin/env python3
"""Summarise an ncu report: key metrics + top source lines by stall samples and by instructions."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]} {rows[1][h.index(k)]}")
for k, x in zip(h, v):
    if "warps_issue_stalled" in k and k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
        try:
            if float(x) > 0.05:
                print(f"  {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio',''):30s} {float(x):.3f}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
res = collections.defaultdict(lambda: [0, 0]); cur = None; curline = None
for r in csv.reader(src.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) > 7 and r[0] not in ("", "Function Name", "Line No") and r[2] == "-":
        curline = (cur, r[0], r[1][:80])
        res[curline][0] += int(r[4] or 0); res[curline][1] += int(r[7] or 0)
tw = sum(x[0] for x in res.values()) or 1; te = sum(x[1] for x in res.values()) or 1
print("top lines by stall samples (samples%, inst%)")
for k, x in sorted(res.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{x[0]/tw*100:5.1f}% {x[1]/te*100:5.1f}%  {k[0]}:{k[1]} {k[2]}")
