"""Per-iteration re-scoring counts and step times of the bench workload
(config 3 by default): scores the scorer flagged and listed for the
one-component tensor pass, scores still flagged and re-evaluated in fp64, and
the graphed step time. Usage: python tools/dbg/fix_counts.py [iters] [bench args]"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import bench  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402
from paper_2501_12299_b200.sharded import Comm  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sys.argv = [sys.argv[0]] + sys.argv[2:]
args = bench.parse()
comm = Comm(device="cuda:0")
m, X, p, st, floor, a, b, n_total = bench.build_problem(V, args, 0, 1, comm)
C, H, Cp, G = m["C"], m["H"], m["Cprime"], m["G"]
sess = V.Session(C, X.shape[1], H, Cp, G, X, n_offset=a, n_total=n_total, device=0)
sess.set_floor(floor)
sess.upload_params(p)
sess.upload_state(st)
ext = torch.cuda.ExternalStream(sess.stream())
for it in range(2):
    sess.variational_e_step(0, it)
w = sess.scoring_work()
print(f"warm E-steps: listed {w['tensor_rescored']} fp64 {w['fp64_rescored']}", flush=True)
for it in range(2, 2 + iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    r = sess.iterate(0, it)
    e1.record(ext)
    e1.synchronize()
    w = sess.scoring_work()
    print(f"it {it:3d}: {e0.elapsed_time(e1):7.2f} ms  joints {r['joints']:.4g}  listed {w['tensor_rescored']:9d}"
          f"  fp64 {w['fp64_rescored']:8d}  F {r['F']:.10g}", flush=True)
