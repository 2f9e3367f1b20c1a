"""Phase timing of k_stats on CTA 0 (diagnostics; vmfa_diag_stats_cycles).

Needs a library built with the marks compiled in:
    VMFA_NVCC_EXTRA=-DVMFA_STATS_PROF python -c "from paper_2501_12299_b200 import build as B; B.build(force=True)"
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2501_12299_b200 import vmfa as V  # noqa: E402
from paper_2501_12299_b200.abi import lib  # noqa: E402

X = V.gen_synthetic(V.synth_spec(2))
m = V.CONFIGS[2]["model"]
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
for it in range(2):
    s.variational_e_step(0, it)
for it in range(2, 5):
    s.iterate(0, it)
L = lib()
f = L.vmfa_diag_stats_cycles
f.restype = C.c_int
f.argtypes = [C.c_int, C.c_void_p]
out = np.zeros(16, np.uint64)
f(1, None)
s.variational_e_step(0, 10)
import time
s.accumulate_suffstats()
f(1, out.ctypes.data_as(C.c_void_p))
f(0, None)
names = ["", "-", "wait rows", "-", "phase i", "sync A", "z reduce", "sync B", "E + phase ii", "issue"]
tot = out[1:10].sum()
for i in range(1, 10):
    print(f"{names[i]:18s} {int(out[i]):12d} {100 * out[i] / tot:5.1f}%")
