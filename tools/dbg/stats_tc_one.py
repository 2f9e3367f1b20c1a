"""Debug: one statistics pass on the tcgen05 kernel, small shape, timed."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
from _helpers import gaussian_problem, to_vmfa_params, to_vmfa_state  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

N, D, C, H, Cp, G = [int(v) for v in (sys.argv[1:] or [2000, 64, 8, 3, 2, 3])]
X, _ = gaussian_problem(N, D, max(2, C // 2), min(H, 4), seed=5)
p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
sess = V.Session(C, D, H, Cp, G, X)
sess.set_floor(floor)
sess.upload_params(to_vmfa_params(V, p))
sess.upload_state(to_vmfa_state(V, st))
sess.variational_e_step(0, 0)
_, _, _, resp = sess.download_estep()
stg = sess.download_state()
t = time.time()
try:
    sess.accumulate_suffstats()
    print("ok", time.time() - t)
except Exception as e:
    print("fail after", time.time() - t, e)
    raise
s = sess.download_suffstats()
k = O.precompute_all(p)
so = O.accumulate_suffstats(X, p, k, stg.K, resp, threads=4)
for f in ("Nc", "E", "Y", "sq"):
    a, b = getattr(s, f), getattr(so, f)
    print(f, float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)))
for f in ("E", "Y", "sq"):
    a, b = getattr(s, f).reshape(C, -1), getattr(so, f).reshape(C, -1)
    r = np.abs(a - b).max(1) / np.maximum(np.abs(b).max(1), 1e-300)
    w = int(np.argmax(r))
    print(f, "per-comp worst", float(r[w]), "comp", w, "Nc", float(so.Nc[w]))
    if f == "Y":
        yy = np.abs(a[w] - b[w]).reshape(H + 1, D)
        print("   worst (h,d)", np.unravel_index(np.argmax(yy), yy.shape), "rel per h", (yy.max(1) / np.maximum(np.abs(b[w].reshape(H + 1, D)).max(1), 1e-300)).round(8))
