"""Diagnostics for the scale parity tests: one teacher-forced run, every
check recorded instead of asserted; prints the worst log-joint rows and the
worst parameter components with their statistics."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402
from _helpers import to_vmfa_params, to_vmfa_state  # noqa: E402

cfg = int(sys.argv[1])
N = int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
X = V.gen_synthetic(V.synth_spec(cfg), 0, N)
m = V.CONFIGS[cfg]["model"]
C, H, Cp, G = m["C"], m["H"], m["Cprime"], m["G"]
T = os.cpu_count()
p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
sess = V.Session(C, X.shape[1], H, Cp, G, X)
sess.set_floor(floor)
for it in range(iters):
    k = O.precompute_all(p)
    sess.upload_params(to_vmfa_params(V, p))
    st_or = st.copy()
    e = O.variational_e_step(X, p, k, st_or, 0, it, threads=T)
    sess.upload_state(to_vmfa_state(V, st))
    F, J = sess.variational_e_step(0, it)
    print(f"   fp64 rescored: {sess.scoring_work()['fp64_rescored']}")
    cnt, idx, lj, resp = sess.download_estep()
    fin = np.isfinite(e.lj) & (idx >= 0)
    err = np.where(fin, np.abs(lj - e.lj), 0)
    rel = err / np.maximum(np.abs(e.lj), 1.0)
    # error against the magnitude of the log-joint's terms (model.cpp:87-94):
    # |log pi| + 0.5 (D log 2pi + |log|Sigma|| + Q), Q = the Mahalanobis term
    kk = O.precompute_all(p)
    cc = np.where(idx >= 0, idx, 0)
    lpi = kk.log_pi[cc]
    ld = kk.logdet[cc]
    Dl = X.shape[1] * 1.8378770664093453
    Q = -2.0 * (e.lj - lpi) - Dl - ld
    scale = np.abs(lpi) + 0.5 * (Dl + np.abs(ld) + np.abs(Q))
    relm = np.where(fin, err / scale, 0)
    print(f"   M-scale rel max {relm.max():.3e}, rows>1e-4 {(relm.max(1) > 1e-4).sum()}; abs err max {err.max():.3g}")
    Lnorm = np.sqrt((kk.Lmat.reshape(C, -1) ** 2).sum(1))
    fl = np.min(p.psi / floor[None, :], axis=1)
    badm = relm > 1e-4
    if badm.any():
        bc = np.unique(idx[badm])
        print(f"   M-bad pairs {badm.sum()} in {len(bc)} comps; their |L|_F min/med {Lnorm[bc].min():.3g}/{np.median(Lnorm[bc]):.3g}"
              f", psi_min/floor min/med/max {fl[bc].min():.3g}/{np.median(fl[bc]):.3g}/{fl[bc].max():.3g}")
    for thr in (1e2, 1e3, 1e4, 1e5):
        flag = Lnorm > thr
        fp = flag[cc] & fin
        print(f"   |L|_F>{thr:g}: {flag.sum()} comps, {fp.sum()} pairs ({fp.sum() / fin.sum():.3%}); M-bad left {(badm & ~fp).sum()}")
    print(f"   |L|_F quantiles all comps: {np.quantile(Lnorm, [0.5, 0.9, 0.99, 1.0])}")
    n, j = np.unravel_index(np.argmax(rel), rel.shape)
    c = idx[n, j]
    print(f"it {it}: J {J} vs {e.joints}, F rel {abs(F - e.F) / abs(e.F):.2e}, lj rel max {rel.max():.3e} "
          f"(n={n} c={c} lj_or={e.lj[n, j]:.6g} gpu={lj[n, j]:.6g}), rows>1e-4: {(rel.max(1) > 1e-4).sum()}")
    bad_c = np.unique(idx[rel > 1e-4])
    print("   components with rel>1e-4:", len(bad_c), bad_c[:10])
    for c in bad_c[:5]:
        d = np.linalg.norm(p.mu[c] - X[n]) if True else 0
        print(f"   c={c} pi={p.pi[c]:.3g} psi[min,max]=[{p.psi[c].min():.3g},{p.psi[c].max():.3g}] "
              f"|lam|max={np.abs(p.lam[c]).max():.3g} |mu|max={np.abs(p.mu[c]).max():.3g}")
    # anchors of the worst row
    print("   worst row K:", st.K[n], "psi min of anchors:", [float(p.psi[a].min()) for a in st.K[n]])
    st_g = sess.download_state()
    sess.accumulate_suffstats()
    s_g = sess.download_suffstats()
    s_or = O.accumulate_suffstats(X, p, k, st_g.K, resp, threads=T)
    for f in ("Nc", "E", "Y", "sq"):
        a, b = getattr(s_g, f), getattr(s_or, f)
        a2, b2 = a.reshape(C, -1), b.reshape(C, -1)
        r = np.abs(a2 - b2).max(1) / np.maximum(np.abs(b2).max(1), 1e-300)
        w = np.argmax(r)
        print(f"   stats {f}: per-comp rel max {r.max():.3e} at c={w} (Nc={s_or.Nc[w]:.3g}), q999 {np.quantile(r, .999):.3e}")
    sess.update_params()
    p_g = sess.download_params()
    p_or = O.update_params(s_or, N, p, floor)
    for f in ("pi", "mu", "lam", "psi"):
        a, b = getattr(p_g, f), getattr(p_or, f)
        a2, b2 = a.reshape(C, -1), b.reshape(C, -1)
        r = np.abs(a2 - b2).max(1) / np.maximum(np.abs(b2).max(1), 1e-300)
        w = np.argmax(r)
        print(f"   param {f}: rel max {r.max():.3e} at c={w} Nc={s_or.Nc[w]:.3g} |b|max={np.abs(b2[w]).max():.3g}"
              f" q999 {np.quantile(r, .999):.3e}; comps>1e-3: {(r > 1e-3).sum()}")
        if f == "lam" and r.max() > 1e-2:
            E = s_or.E[w]
            print("     E eig:", np.linalg.eigvalsh(E)[:4], "Nc", s_or.Nc[w], "gpu E eig", np.linalg.eigvalsh(s_g.E[w])[:4])
    Fp = sess.truncated_free_energy()
    Fo = O.truncated_free_energy(X, p_or, O.precompute_all(p_or), st_g.K, threads=T)
    print(f"   F post rel {abs(Fp - Fo) / abs(Fo):.2e}")
    p, st = p_or, st_or
