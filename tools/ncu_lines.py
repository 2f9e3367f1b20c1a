"""Warp-stall samples aggregated per CUDA source line (ncu --page source, cuda,sass)."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
stall = [i for i, x in enumerate(h) if x.startswith("stall_")]
agg, src, why = defaultdict(float), {}, defaultdict(lambda: defaultdict(float))
line = None
for r in rows[hi + 1:]:
    if len(r) <= si:
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        line = int(r[0])
        src[line] = r[1]
    try:
        v = float(r[si])
    except ValueError:
        continue
    agg[line] += v
    for i in stall:
        try:
            why[line][h[i]] += float(r[i])
        except ValueError:
            pass
tot = sum(agg.values())
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:ntop]:
    top = sorted(why[ln].items(), key=lambda x: -x[1])[:2]
    print(f"{ln:5d} {100 * v / tot:5.1f}%  {src.get(ln, '')[:80]:80s} " + " ".join(f"{k[6:]}:{100 * w / max(v, 1):.0f}%" for k, w in top))
