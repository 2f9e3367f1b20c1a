"""Full-size parity evidence on BASELINE config 2 (N = 200 000, D = 256,
C = 1000, H = 8, C' = 5, G = 10): the device and the fp64 oracle run the same
seeded data and initialisation side by side, 2 warm-up E-steps then main
iterations, (a) free-running and (b) teacher-forced (the device restarts each
iteration from the oracle's parameters and state). Reports, per iteration,
the joint counts, the E-step free energy, the post-M-step free energy and
their relative differences (north star: 1e-4), plus the K-row agreement.
Takes a few minutes of host time: python tools/parity_config2.py [iters]."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
threads = os.cpu_count() or 8
m = V.CONFIGS[2]["model"]
C, H, Cp, G = m["C"], m["H"], m["Cprime"], m["G"]
X = V.gen_synthetic(V.synth_spec(2))
N = X.shape[0]
p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
print(f"config 2: N={N} D={X.shape[1]} C={C} H={H} C'={Cp} G={G}; oracle threads={threads}", flush=True)


def session(p, st):
    s = V.Session(C, X.shape[1], H, Cp, G, X)
    s.set_floor(floor)
    s.upload_params(V.Params(p.pi, p.mu, p.lam, p.psi))
    s.upload_state(V.State(st.K, st.g, st.g_count))
    return s


for mode in ("free-running", "teacher-forced"):
    po, so = O.Params(p.pi.copy(), p.mu.copy(), p.lam.copy(), p.psi.copy()), st.copy()
    s = session(po, so)
    k = O.precompute_all(po)
    it = 0
    for _ in range(2):  # warm-up E-steps
        Fg, Jg = s.variational_e_step(0, it)
        e = O.variational_e_step(X, po, k, so, 0, it, threads=threads)
        print(f"[{mode}] warm-up {it}: joints {Jg} vs {e.joints}; F_estep {Fg:.6f} vs {e.F:.6f} "
              f"(rel {abs(Fg - e.F) / abs(e.F):.2e})", flush=True)
        it += 1
    for _ in range(iters):
        if mode == "teacher-forced":
            s.upload_params(V.Params(po.pi, po.mu, po.lam, po.psi))
            s.upload_state(V.State(so.K, so.g, so.g_count))
        t0 = time.perf_counter()
        r = s.iterate(0, it)
        tg = time.perf_counter() - t0
        t0 = time.perf_counter()
        e = O.variational_e_step(X, po, k, so, 0, it, threads=threads)
        S = O.accumulate_suffstats(X, po, k, so.K, e.resp, threads=threads)
        po = O.update_params(S, N, po, floor)
        k = O.precompute_all(po)
        F = O.truncated_free_energy(X, po, k, so.K, threads=threads)
        to = time.perf_counter() - t0
        Kg = s.download_state().K
        same = float(np.mean(np.all(Kg == so.K, axis=1)))
        print(f"[{mode}] iteration {it}: joints {r['joints']} vs {e.joints}; "
              f"F_estep rel {abs(r['F_estep'] - e.F) / abs(e.F):.2e}; F {r['F']:.6f} vs {F:.6f} "
              f"(rel {abs(r['F'] - F) / abs(F):.2e}); K rows identical {same:.5f}; "
              f"device {tg * 1e3:.1f} ms (wall, incl. sync) vs oracle {to:.1f} s", flush=True)
        it += 1
    s.close()
