"""Config-5 model shape, free-running on the GPU; when an update or
precompute fails, the oracle redoes that update from the GPU's own statistics
and previous parameters (diagnostics: which side produces the non-finite /
non-PD component)."""
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
for it in range(2):
    s.variational_e_step(0, it)
use_iterate = len(sys.argv) > 3 and sys.argv[3] == "iterate"
for it in range(2, 30):
    if use_iterate:
        try:
            s.iterate(0, it)
            print(it, "iterate ok", flush=True)
            continue
        except Exception as ex:  # noqa: BLE001
            print(it, "iterate raised:", ex, flush=True)
            break
    prev = s.download_params()
    s.variational_e_step(0, it)
    s.accumulate_suffstats()
    try:
        s.update_params()
        print(it, "ok", flush=True)
        continue
    except Exception as ex:  # noqa: BLE001
        err = str(ex)
        print(it, "gpu update/precompute raised:", ex, flush=True)
    if C > 5000:  # one component's statistics through the exchange buffer (the whole set is ~20 GB)
        import torch
        from paper_2501_12299_b200.exchange import device_view
        ptr, n, _ = s.exchange_buffer(1)
        buf = device_view(ptr, n, "<f8")
        c = int(err.split()[-1])
        D, H1 = X.shape[1], H + 1
        Nc = buf[c].item()
        E = buf[C + c * H1 * H1: C + (c + 1) * H1 * H1].cpu().numpy().reshape(1, H1, H1)
        Y = buf[C + C * H1 * H1 + c * H1 * D: C + C * H1 * H1 + (c + 1) * H1 * D].cpu().numpy().reshape(1, H1, D)
        off = C + C * H1 * H1 + C * H1 * D
        sq = buf[off + c * D: off + (c + 1) * D].cpu().numpy().reshape(1, D)
        print("  comp", c, "N_c", Nc, "E finite", np.isfinite(E).all(), "Y finite", np.isfinite(Y).all(),
              "sq finite", np.isfinite(sq).all(), flush=True)
        ev = np.linalg.eigvalsh(0.5 * (E[0] + E[0].T))
        print("  E eigenvalues min/max", ev.min(), ev.max(), flush=True)
        S1 = O.Stats(np.array([Nc]), Y, E, sq)
        prev1 = O.Params(np.ones(1), np.zeros((1, D)), np.zeros((1, H, D)), np.ones((1, D)))
        try:
            p1 = O.update_params(S1, N, prev1, floor)
            print("  oracle update: psi min/max", p1.psi.min(), p1.psi.max(), "lam max", np.abs(p1.lam).max(),
                  "finite", np.isfinite(p1.lam).all(), flush=True)
            O.precompute_all(p1)
            print("  oracle update + precompute from the GPU statistics of this component: ok", flush=True)
        except Exception as ex2:  # noqa: BLE001
            print("  oracle from the GPU statistics raised:", ex2, flush=True)
        break
    S = s.download_suffstats()
    comp = [c for c in range(C) if not (np.isfinite(S.Y[c]).all() and np.isfinite(S.E[c]).all()
                                        and np.isfinite(S.sq[c]).all())]
    print("  non-finite statistics in", comp[:10], flush=True)
    po = O.Params(prev.pi.copy(), prev.mu.copy(), prev.lam.copy(), prev.psi.copy())
    try:
        p2 = O.update_params(S, N, po, floor)
        O.precompute_all(p2)
        print("  oracle update + precompute from the GPU statistics: ok", flush=True)
    except Exception as ex:  # noqa: BLE001
        print("  oracle from the GPU statistics raised:", ex, flush=True)
    break
