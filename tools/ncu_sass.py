"""Top SASS instructions by warp-stall samples from an ncu report, with the
dominant stall reasons:  python tools/ncu_sass.py report.ncu-rep [N] [--ctx K]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
args = [a for a in sys.argv[2:] if not a.startswith("--")]
n = int(args[0]) if args else 40
ctx = int(sys.argv[sys.argv.index("--ctx") + 1]) if "--ctx" in sys.argv else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, hdr = [], None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    rows.append(r)
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[col["# Samples"]] or 0) for r in rows) or 1
print("total samples", tot)
idx = sorted(range(len(rows)), key=lambda i: -float(rows[i][col["# Samples"]] or 0))[:n]
for i in idx:
    r = rows[i]
    s = float(r[col["# Samples"]] or 0)
    top = sorted(((float(r[col[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    why = " ".join(f"{h}={int(v)}" for v, h in top if v > 0)
    print(f"{100 * s / tot:5.1f}% #{i:5d} ex={r[col['Instructions Executed']]:>8s} {r[col['Source']].strip()[:70]:70s} {why}")
    for j in range(max(0, i - ctx), min(len(rows), i + ctx + 1)):
        if ctx and j != i:
            print(f"        #{j:5d} {rows[j][col['Source']].strip()[:90]}")
