"""Diagnostic: log-joint error of the tcgen05 and FFMA scorers vs the fp64 oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from _helpers import gaussian_problem, to_vmfa_params, to_vmfa_state  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

for case in [dict(N=4000, D=256, C=200, H=8, Cp=5, G=10), dict(N=4000, D=64, C=100, H=4, Cp=3, G=5)]:
    X, _ = gaussian_problem(case["N"], case["D"], case["C"] // 2, min(case["H"], 4), seed=7)
    C, H, Cp, G = case["C"], case["H"], case["Cp"], case["G"]
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    st_or = st.copy()
    e = O.variational_e_step(X, p, k, st_or, 11, 0, threads=8)
    for sc in ("ffma", "tc"):
        os.environ["VMFA_SCORER"] = sc
        s = V.Session(C, X.shape[1], H, Cp, G, X)
        s.set_floor(floor)
        s.upload_params(to_vmfa_params(V, p))
        s.upload_state(to_vmfa_state(V, st))
        s.variational_e_step(11, 0)
        cnt, idx, lj, resp = s.download_estep()
        live = e.idx >= 0
        err = np.abs(lj - e.lj)[live]
        rel = err / np.maximum(1, np.abs(e.lj[live]))
        print(case, sc, "abs max %.3e p99 %.3e mean %.3e | rel max %.3e | |l| median %.1f" %
              (err.max(), np.quantile(err, 0.99), err.mean(), rel.max(), np.median(np.abs(e.lj[live]))))
        worst = np.argmax(np.abs(lj - e.lj) * live)
        print("   worst at", np.unravel_index(worst, lj.shape), lj.flat[worst], e.lj.flat[worst])
        s.close()
