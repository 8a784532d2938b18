"""Per-CUDA-source-line warp stall samples from an ncu report (needs -lineinfo
and --import-source on):  python tools/ncu_src.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, agg = None, None, {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or r[2] != "-":
        continue  # CUDA-line rows carry '-' in the Address column
    try:
        s = float(r[4] or 0)
        ex = float(r[7] or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    a = agg.setdefault(key, [0.0, 0.0, r[1].strip()])
    a[0] += s
    a[1] += ex
tot = sum(v[0] for v in agg.values()) or 1
print("samples", tot)
for (f, ln), (s, ex, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * s / tot:5.1f}% {ex:9.0f} {f}:{ln:5s} {src[:90]}")
