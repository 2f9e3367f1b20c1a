"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel name, launches and total / per-launch time over the last `k`
launches of each name (steady state), and the share of the total."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
by = defaultdict(list)
for r in rows:
    name = r[4].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    by[name].append(float(r[-1]) / 1e3)  # us
tot = sum(sum(v[-last:] if last else v) for v in by.values())
for name, v in sorted(by.items(), key=lambda kv: -sum(kv[1][-last:] if last else kv[1])):
    u = v[-last:] if last else v
    print(f"{sum(u):10.1f} us {100 * sum(u) / tot:5.1f}%  n={len(u):4d}  mean={sum(u) / len(u):9.1f} us  {name[:90]}")
