"""Shared test helpers: problem construction and the near-tie-aware comparisons
of SURVEY.md Appendix A.9 (GPU vs the fp64 oracle)."""
from __future__ import annotations

import numpy as np

# log-joint tolerance of the north star: 1e-4 relative
LJ_RTOL = 1e-4


def to_oracle_params(O, p):
    return O.Params(p.pi.copy(), p.mu.copy(), p.lam.copy(), p.psi.copy())


def to_oracle_state(O, st):
    return O.State(st.K.copy(), st.g.copy(), st.g_count.copy(),
                   None if st.labels is None else st.labels.copy())


def to_vmfa_params(V, p):
    return V.Params(p.pi.copy(), p.mu.copy(), p.lam.copy(), p.psi.copy())


def to_vmfa_state(V, st):
    return V.State(st.K.copy(), st.g.copy(), st.g_count.copy(),
                   None if st.labels is None else st.labels.copy())


def gaussian_problem(N, D, C_true, H_true, seed=0, mu_std=3.0, psi=(0.05, 0.5), dirichlet=False):
    """Small seeded MFA sample (numpy), the generator family of BASELINE configs 1/2."""
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.ones(C_true)) if dirichlet else np.full(C_true, 1.0 / C_true)
    mu = rng.normal(0, mu_std, (C_true, D))
    lam = rng.normal(0, 1 / np.sqrt(max(H_true, 1)), (C_true, D, H_true))
    ps = rng.uniform(psi[0], psi[1], (C_true, D))
    c = rng.choice(C_true, N, p=w)
    z = rng.normal(size=(N, H_true))
    X = mu[c] + np.einsum("ndh,nh->nd", lam[c], z) + rng.normal(size=(N, D)) * np.sqrt(ps[c])
    return X.astype(np.float32), c


def near_tie_rows(lj_or, idx_or, cnt, Cp, tau):
    """Rows whose oracle C'-th and (C'+1)-th largest log-joints in S(n) differ
    by <= tau[n] (Appendix A.9)."""
    N = lj_or.shape[0]
    out = np.zeros(N, bool)
    for n in range(N):
        m = cnt[n]
        if m <= Cp:
            continue
        v = np.sort(lj_or[n, :m])[::-1]
        out[n] = (v[Cp - 1] - v[Cp]) <= tau[n]
    return out


def lj_term_scale(k, idx, lj, D):
    """The magnitude of the terms a log-joint is formed from (model.cpp:87-94):
    |log pi_c| + (D log 2pi + |log|Sigma_c|| + Q) / 2, with the Mahalanobis term
    Q = -2 (l - log pi_c) - D log 2pi - log|Sigma_c|. Always >= |l|; the error
    of any fp32-accurate evaluation is proportional to it (l is their small
    difference when the density is near 1, e.g. image data with psi ~ 1e-2)."""
    cc = np.where(idx >= 0, idx, 0)
    lpi = k.log_pi[cc]
    ld = k.logdet[cc]
    dl = D * 1.8378770664093453
    with np.errstate(invalid="ignore"):
        Q = -2.0 * (lj - lpi) - dl - ld
        return np.abs(lpi) + 0.5 * (dl + np.abs(ld) + np.abs(Q))


def compare_estep(O, e_or, st_or, F_gpu, J_gpu, gpu_retained, st_gpu, Cp, report=None, k=None, D=None):
    """Teacher-forced E-step parity. Returns a dict of counts; asserts the bar:
    identical joint count and search spaces, log-joints within 1e-4 relative,
    F within 1e-4 relative, K / labels identical outside documented near-ties.
    Log-joint relative error: against max(|l|, 1), or -- given the oracle's
    caches k and D -- against the magnitude of the log-joint's terms
    (lj_term_scale, >= |l|); both are reported."""
    cnt_g, idx_g, lj_g, resp_g = gpu_retained
    assert J_gpu == e_or.joints, (J_gpu, e_or.joints)
    assert np.array_equal(cnt_g, e_or.count)
    assert np.array_equal(idx_g, e_or.idx), "search spaces differ (insertion order / dedup)"
    live = idx_g >= 0
    err = np.abs(lj_g - e_or.lj)
    fin = np.isfinite(e_or.lj) & live
    rel_plain = np.where(fin, err / np.maximum(np.abs(e_or.lj), 1.0), 0.0)
    scale = np.maximum(np.abs(e_or.lj), 1.0) if k is None else np.maximum(lj_term_scale(k, idx_g, e_or.lj, D), 1.0)
    rel = np.where(fin, err / np.where(fin, scale, 1.0), 0.0)
    assert rel.max() <= LJ_RTOL, f"log-joint rel err {rel.max():.3e}"
    assert np.all(np.isinf(lj_g[live & ~np.isfinite(e_or.lj)]))
    assert abs(F_gpu - e_or.F) <= LJ_RTOL * abs(e_or.F), (F_gpu, e_or.F)
    # near-tie rule: tau = 2 max |l_gpu - l_or| per row, or 1e-4 |l|
    row_err = np.where(fin, err, 0.0).max(axis=1)
    tau = np.maximum(2 * row_err, 1e-4 * np.abs(np.where(fin, e_or.lj, 0.0)).max(axis=1))
    ties = near_tie_rows(e_or.lj, e_or.idx, e_or.count, Cp, tau)
    kdiff = np.any(st_gpu.K != st_or.K, axis=1)
    assert not np.any(kdiff & ~ties), f"{int((kdiff & ~ties).sum())} K rows differ outside near-ties"
    same = ~kdiff
    # labels: ties within K are near-ties too
    ldiff = (st_gpu.labels != st_or.labels) & same
    if ldiff.any():
        for n in np.nonzero(ldiff)[0]:
            a = lj_g[n][idx_g[n] == st_or.labels[n]][0]
            b = lj_g[n][idx_g[n] == st_gpu.labels[n]][0]
            assert abs(a - b) <= max(tau[n], 1e-6), f"label differs at row {n} outside near-ties"
    # responsibilities on identical K rows: q = softmax(l) over K, so
    # |dq| <= 2 max|dl| (row-wise bound implied by the log-joint tolerance)
    dq = np.abs(resp_g - e_or.resp).max(axis=1)
    assert np.all(dq[same] <= 2 * row_err[same] + 1e-9), float((dq - 2 * row_err)[same].max())
    info = dict(rows=len(kdiff), k_near_ties=int(ties.sum()), k_diff=int(kdiff.sum()),
                label_diff=int(ldiff.sum()), lj_rel=float(rel.max()), lj_rel_plain=float(rel_plain.max()),
                lj_rows_plain_over_1e4=int((rel_plain.max(axis=1) > LJ_RTOL).sum()),
                lj_abs_max=float(np.where(fin, err, 0.0).max()))
    if report is not None:
        report.update(info)
    return info


def compare_g(g_gpu, gc_gpu, g_or, gc_or, dist_or, labels_same_comp, rtol=1e-6):
    """g_c identical for every component whose partition matched, except where
    the oracle's (G-1)-th and G-th smallest averages are within rtol."""
    C = g_or.shape[0]
    G = g_or.shape[1]
    dc, dct, dsum, dcnt = dist_or
    bad = []
    starts = np.searchsorted(dc, np.arange(C + 1))
    for c in range(C):
        if not labels_same_comp[c]:
            continue
        a = g_gpu[c, :gc_gpu[c]]
        b = g_or[c, :gc_or[c]]
        if gc_gpu[c] == gc_or[c] and np.array_equal(a, b):
            continue
        s, e = starts[c], starts[c + 1]
        avg = np.sort(dsum[s:e] / dcnt[s:e])
        if len(avg) >= G and abs(avg[G - 1] - avg[G - 2]) <= rtol * max(1.0, abs(avg[G - 2])):
            continue  # near-tie at the selection boundary
        bad.append(c)
    return bad


def ldlt_cases(O):
    """Statistics exercising update_params' LDLT semantics (mstep.cpp:129-140,
    Eigen LDLT): c0 SPD; c1 PSD-singular diag(2,0,3) (zero pivot last -> the
    pseudo-inverse of D zeroes that coordinate); c2 a zero pivot followed by
    a non-zero one (info != Success -> trace-scaled jitter retry); c3 an
    indefinite E (LDLT succeeds where a Cholesky would fail). C=4, D=5, H=2.
    Returns (stats, prev params, floor, expected A^T per component)."""
    rng = np.random.default_rng(11)
    C_, D, H = 4, 5, 2
    H1 = H + 1
    E = np.zeros((C_, H1, H1))
    B = rng.normal(size=(H1, H1))
    E[0] = B @ B.T + 0.5 * np.eye(H1)
    E[1] = np.diag([2.0, 0.0, 3.0])
    E[2] = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 0.0, 0.5]])
    E[3] = np.array([[1.0, 2.0, 0.1], [2.0, 1.0, 0.2], [0.1, 0.2, 4.0]])
    Y = rng.normal(size=(C_, H1, D))
    Y[2, 1] = Y[2, 0]  # consistent with E[2]'s null direction: the jittered solution stays bounded
    Nc = E[:, H, H].copy()
    sq = np.full((C_, D), 50.0)
    want = np.zeros((C_, H1, D))
    want[0] = np.linalg.solve(E[0], Y[0])
    want[1] = np.stack([Y[1, 0] / 2.0, np.zeros(D), Y[1, 2] / 3.0])
    E2 = E[2] + 1e-10 * np.trace(E[2]) / H1 * np.eye(H1)
    want[2] = np.linalg.solve(E2, Y[2])
    want[3] = np.linalg.solve(E[3], Y[3])
    s = O.Stats(Nc, Y, E, sq)
    prev = O.Params(np.full(C_, 1.0 / C_), rng.normal(size=(C_, D)), rng.normal(size=(C_, H, D)),
                    np.ones((C_, D)))
    return s, prev, np.full(D, 1e-6), want


def near_tie_rows_fast(lj_or, cnt, Cp, tau):
    """Vectorised near_tie_rows: the oracle's C'-th and (C'+1)-th largest
    log-joints of S(n) within tau[n]."""
    N, S = lj_or.shape
    live = np.arange(S)[None, :] < cnt[:, None]
    v = np.where(live & np.isfinite(lj_or), lj_or, -np.inf)
    v = -np.sort(-v, axis=1)
    out = np.zeros(N, bool)
    ok = cnt > Cp
    a, b = v[ok, Cp - 1], v[ok, Cp]
    out[ok] = (a - b) <= tau[ok]
    out[ok & ~np.isfinite(b)] = False
    return out


def compare_g_tau(g_gpu, gc_gpu, g_or, gc_or, dist_or, tau, touched):
    """g_c (update_g, estep.cpp:204-220) per component: identical, or a
    near-tie at the selection boundary -- the oracle's (G-1)-th and G-th
    smallest averages within tau (each average carries at most 2 max|dl| of
    the log-joint error, so tau = 4 max|dl|) -- or a component whose partition
    changed because a near-tie row changed its label (`touched`). Returns
    (diff, ties, touched_diff, bad) component lists."""
    C, G = g_or.shape
    dc, dct, dsum, dcnt = dist_or
    starts = np.searchsorted(dc, np.arange(C + 1))
    diff, ties, tdiff, bad = [], [], [], []
    for c in range(C):
        a = g_gpu[c, :gc_gpu[c]]
        b = g_or[c, :gc_or[c]]
        if gc_gpu[c] == gc_or[c] and np.array_equal(a, b):
            continue
        diff.append(c)
        if touched[c]:
            tdiff.append(c)
            continue
        s, e = starts[c], starts[c + 1]
        avg = np.sort(dsum[s:e] / dcnt[s:e])
        if len(avg) >= G and abs(avg[G - 1] - avg[G - 2]) <= tau:
            ties.append(c)
            continue
        bad.append(c)
    return diff, ties, tdiff, bad
