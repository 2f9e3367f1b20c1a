"""Top SASS instructions by warp-stall samples from an ncu report (--page source)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
stall = [i for i, x in enumerate(h) if x.startswith("stall_")]


def num(x):
    try:
        return float(x)
    except ValueError:
        return None


data = [r for r in rows[2:] if len(r) > si and num(r[si]) is not None]
tot = sum(num(r[si]) for r in data)
print("total samples", tot, "instructions", len(data))
agg = {}
for r in data:
    for i in stall:
        agg[h[i]] = agg.get(h[i], 0) + (num(r[i]) or 0)
print(" ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:12]))
top = sorted(range(len(data)), key=lambda k: -num(data[k][si]))[:ntop]
for k in sorted(top):
    r = data[k]
    st = sorted(((num(r[i]) or 0, h[i][6:]) for i in stall), reverse=True)[:2]
    print(f"{k:5d} {r[1][:64]:64s} {100 * num(r[si]) / tot:5.1f}% " + " ".join(f"{n}:{v:.0f}" for v, n in st))
