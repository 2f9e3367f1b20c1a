"""Summarise ncu outputs brought back by gpurun into profiles/<round>/.

  python tools/summarize_ncu.py --round r01 \
      --launches gpurun_out/r01_launches.csv --full gpurun_out/r01_full.ncu-rep \
      --bench gpurun_out/r01_bench.json

Writes
  profiles/<round>/launches.csv            the raw gpu__time_duration launch list
  profiles/<round>/launch_shares.txt       per-kernel totals and shares of the list
  profiles/<round>/ncu_full_summary.csv    selected --set full metrics per launch
  profiles/<round>/bench.json              the bench line of the same code
  profiles/<round>/scorer_traffic_configN.json  DRAM bytes of one scoring launch
                                           pair (anchor + extra), read by bench.py
                                           for roofline.traffic
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.sum",
    "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def to_us(unit: str, v: str) -> float:
    v = float(v.replace(",", ""))
    return {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
            "s": 1e6, "second": 1e6}[unit] * v


def short(name: str) -> str:
    m = re.search(r"\b(k_\w+(?:<[^>]*>)?)", name)
    if m:  # our kernels: the bare name (+ template arguments)
        return m.group(1)
    return name.replace("void ", "").split("(")[0]


def launch_shares(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ui, vi = h.index("Kernel Name"), h.index("Metric Unit"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        k = short(r[ki])
        tot[k] += to_us(r[ui], r[vi])
        cnt[k] += 1
    T = sum(tot.values())
    out = [f"# {len(rows) - 1} launches, {T:.1f} us total (ncu, serialised, cold cache)",
           f"{'kernel':58s} {'n':>4s} {'total_us':>10s} {'share':>6s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k[:58]:58s} {cnt[k]:4d} {v:10.1f} {100 * v / T:5.1f}%")
    return "\n".join(out) + "\n"


def full_summary(rep: str):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(FULL_METRICS)], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    cols = ["Kernel Name"] + [m for m in FULL_METRICS if m in h]
    out = [cols, [""] + [units[h.index(m)] for m in cols[1:]]]
    for r in rows[2:]:
        out.append([short(r[h.index("Kernel Name")])] + [r[h.index(m)] for m in cols[1:]])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--bench")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--full2", help="a second --set full report (other kernels), appended to the summary")
    a = ap.parse_args()
    d = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(d, exist_ok=True)
    if a.launches:
        shutil.copy(a.launches, os.path.join(d, "launches.csv"))
        open(os.path.join(d, "launch_shares.txt"), "w").write(launch_shares(a.launches))
    if a.bench:
        line = [x for x in open(a.bench).read().splitlines() if x.startswith("{")][-1]
        json.dump(json.loads(line), open(os.path.join(d, "bench.json"), "w"), indent=1)
    if a.full:
        rows = full_summary(a.full)
        if a.full2:
            rows += full_summary(a.full2)[2:]
        with open(os.path.join(d, "ncu_full_summary.csv"), "w", newline="") as f:
            csv.writer(f).writerows(rows)
        # scoring launch pair = the anchor launch (the one writing the lj table,
        # largest) + the extra-candidate launch (smallest) of the same E-step
        h = rows[0]
        sc = [r for r in rows[2:] if r[0].startswith("k_score_ws")]
        if len(sc) >= 2:
            tcol, rcol, wcol = (h.index(m) for m in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                                     "dram__bytes_write.sum"))
            units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rs, ws = units[rows[1][rcol]], units[rows[1][wcol]]  # (read and write may differ in unit)
            mb = lambda r: float(r[rcol]) * rs + float(r[wcol]) * ws  # noqa: E731
            sc.sort(key=lambda r: float(r[tcol]))
            anchor, extra = sc[-1], sc[0]
            traffic = {"kernel": "k_score_ws (anchor + extra launch of one E-step)",
                       "bytes_per_launch_pair": mb(anchor) + mb(extra),
                       "anchor_bytes": mb(anchor), "extra_bytes": mb(extra),
                       "anchor_ms": float(anchor[tcol]), "extra_ms": float(extra[tcol]),
                       "source": f"profiles/{a.round}/ncu_full_summary.csv "
                                 "(dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full)"}
            json.dump(traffic, open(os.path.join(d, f"scorer_traffic_config{a.config}.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
