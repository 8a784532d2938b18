"""Per-item clock table of CTA 0 from a -DHODLR_TC_TRACE run (tools/variants build):
python tools/tctrace_table.py gpurun_out/tctrace.log [first last]"""
import re
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith("TRACE")]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 48)
dumps = defaultdict(list)
for l in lines:
    m = re.match(r"TRACE role (\d+) item (\d+) a (-?\d+) b (-?\d+) c (-?\d+) w (-?\d+)", l)
    r, i, a, b, c, w = map(int, m.groups())
    if i == 0:
        dumps[r].append([])
    dumps[r][-1].append((a, b, c, w))
D = {r: dumps[r][-1] for r in dumps}
t0 = min(x for r in D for row in D[r] for x in row if x > 0)
print("item | conv: rawfull aempty fence stored | prod: rawempty | mma: afull bfull commit | stg: barrier issued bempty fenced")
f = lambda x: f"{x - t0:7d}" if x > 0 else "      -"
for i in range(lo, hi):
    c, p, m, s = D[0][i], D[1][i], D[2][i], D[3][i]
    print(f"{i:3d} | {f(c[0])} {f(c[1])} {f(c[2])} {f(c[3])} | {f(p[3])} | {f(m[0])} {f(m[1])} {f(m[2])} | {f(s[3])} {f(s[0])} {f(s[1])} {f(s[2])}")
