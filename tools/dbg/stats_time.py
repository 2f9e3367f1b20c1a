"""Debug: time the statistics pass at a config-3-like shape (synthetic K/resp)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

N, D, C, H, Cp = [int(v) for v in (sys.argv[1:] or [200000, 784, 800, 16, 5])]
X = V.gen_synthetic(V.synth_spec(3, N=N))[:, :D].copy()
p, st, floor, _ = V.initialize(X, C, H, Cp, 10 if C >= 10 else C, seed=0)
sess = V.Session(C, D, H, Cp, 10 if C >= 10 else C, X)
sess.set_floor(floor)
sess.upload_params(p)
sess.upload_state(st)
sess.variational_e_step(0, 0)
for i in range(3):
    t = time.perf_counter()
    sess.accumulate_suffstats()
    print("stats", (time.perf_counter() - t) * 1e3, "ms")
