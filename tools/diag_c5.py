"""Config-5 model shape at a small scale: GPU iterations next to the oracle
(diagnostics for the H = 64 path)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 500
H, Cp, G = 64, 5, 20
X = V.gen_synthetic(V.synth_spec(5), 0, N)
p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
s = V.Session(C, X.shape[1], H, Cp, G, X)
s.set_floor(floor)
s.upload_params(V.Params(p.pi, p.mu, p.lam, p.psi))
s.upload_state(V.State(st.K, st.g, st.g_count))
k = O.precompute_all(p)
for it in range(2):
    s.variational_e_step(0, it)
    e = O.variational_e_step(X, p, k, st, 0, it, threads=8)
for it in range(2, 8):
    # teacher-forced: the GPU starts every iteration from the oracle's parameters and state
    s.upload_params(V.Params(p.pi, p.mu, p.lam, p.psi))
    s.upload_state(V.State(st.K, st.g, st.g_count))
    try:
        r = s.iterate(0, it)
        gerr = None
    except Exception as ex:  # noqa: BLE001
        r, gerr = None, ex
    e = O.variational_e_step(X, p, k, st, 0, it, threads=8)
    S = O.accumulate_suffstats(X, p, k, st.K, e.resp, threads=8)
    try:
        p2 = O.update_params(S, N, p, floor)
        k2 = O.precompute_all(p2)
        oerr = None
    except Exception as ex:  # noqa: BLE001
        oerr = ex
    nc = S.Nc
    print(it, "gpu", "ok" if gerr is None else gerr, "| oracle", "ok" if oerr is None else oerr,
          "| Nc min %.3g, #Nc<H %d, psi min %.3g" % (nc[nc > 0].min(), int(((nc > 0) & (nc < H)).sum()),
                                                      p.psi.min()), flush=True)
    if gerr is not None:
        pg = s.download_params()
        bad = [c for c in range(C) if not (np.isfinite(pg.lam[c]).all() and np.isfinite(pg.psi[c]).all())]
        print("  gpu non-finite params in components", bad[:10], flush=True)
        comp = int(str(gerr).split()[-1]) if str(gerr).split()[-1].isdigit() else None
        if comp is not None and oerr is None:
            print("  comp", comp, "Nc", nc[comp], "oracle psi range", p2.psi[comp].min(), p2.psi[comp].max(),
                  "lam max", np.abs(p2.lam[comp]).max(), flush=True)
        break
    if oerr is not None:
        break
    p, k = p2, k2
