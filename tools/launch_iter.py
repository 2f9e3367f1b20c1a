"""Per-kernel times of ONE iteration of an ncu launch list: the launches
between the last two occurrences of a marker kernel (default k_rowmax, one
per E-step), summed by name."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "k_rowmax"
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[-3] == "gpu__time_duration.sum"]
names = [r[4].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "") for r in rows]
idx = [i for i, n in enumerate(names) if n.endswith(marker)]
a, b = idx[-2], idx[-1]
by = defaultdict(list)
for i in range(a, b):
    by[names[i]].append(float(rows[i][-1]) / 1e3)
tot = sum(sum(v) for v in by.values())
print(f"# one iteration: launches {a}..{b - 1} ({b - a} launches), {tot:.1f} us (ncu, serialised, cold cache)")
for name, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v):10.1f} us {100 * sum(v) / tot:5.1f}%  n={len(v):3d}  {name[:90]}")
