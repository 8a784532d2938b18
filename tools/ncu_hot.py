"""Summarise an ncu report: key metrics + hottest SASS lines (stall samples)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread"]
for w in want:
    if w in hdr:
        print(f"{w:60s} {vals[hdr.index(w)]} {rows[1][hdr.index(w)]}")
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
        try:
            if float(vals[i]) > 0.3:
                print(f"  {h[34:-27]:30s} {vals[i]}")
        except ValueError:
            pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iS, iSrc, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
data = []
for idx, r in enumerate(rows[2:]):
    try:
        data.append((float(r[iS] or 0), idx, r[iSrc], r[iex]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print("samples", tot)
for s, idx, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{s / tot * 100:5.1f}% {idx:5d} {ex:>8} {src[:90]}")
