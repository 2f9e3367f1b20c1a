"""Pins of the fp64 oracle (CPU, no GPU):
  * RNG / LSE bit-exact against golden vectors produced by compiling the
    reference's own Eigen-free headers (oracle/ref_golden.cpp ->
    tests/golden/rng_ref.json, rng.hpp:9-98, numerics.hpp:10-22);
  * SPEC.md known-answer examples (SPEC.md:58-60, 68-70, 143-145, 153-155,
    183-185, 193-195, 249-251, 259-261);
  * dense-covariance formulas of proj/tests/oracle.hpp:18-78, reimplemented
    in numpy (acceptance criterion 1);
  * E-step / EM properties of SPEC.md's acceptance criteria 2, 3, 6, 12.
"""
import json
import os

import numpy as np
import pytest

from _helpers import gaussian_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rng_ref.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def _f(v):
    return float(v) if not isinstance(v, str) else float(v.replace("inf", "inf"))


# ------------------------------------------------------------------ reference-compiled pins
def test_uniform_component_matches_reference(oracle, gold):
    for s, it, n, C, r in gold["uniform_component"]:
        assert oracle.uniform_component(int(s), int(it), int(n), C) == r


def test_hashes_match_reference(oracle, gold):
    got = [oracle.hash_combine(a, b) for a in (0, 1, 2, 0xDEADBEEF) for b in (0, 3, 0x1217F01D)]
    assert [str(x) for x in got] == gold["hash_combine_a0_1_2_deadbeef_x_b0_3_1217f01d"]
    got = [oracle.hash3(0, 0, 0), oracle.hash3(1, 2, 3), oracle.hash3(7, 11, 13)]
    assert [str(x) for x in got] == gold["hash3_000_123_71113"]


@pytest.mark.parametrize("salt", [0x1217F01D, 0x7A57A7E5])
def test_trainer_streams_match_reference(oracle, gold, salt):
    got = oracle.rng_u64(oracle.hash_combine(0, salt), 16)
    assert [str(int(x)) for x in got] == gold[f"rng_next_u64_seed0_salt_{salt:x}"]


def test_distributions_match_reference(oracle, gold):
    v = oracle.rng_ops(42, [0] * 9 + [1] + [0] * 6)
    assert np.array_equal(v, np.array(gold["rng42_gaussian9_uniform1_gaussian6"]))  # bit-exact
    b = [1000, 1, 2, 3, 1000000007, 50000000, 100]
    v = oracle.rng_ops(7, [2] * len(b), b)
    assert [str(int(x)) for x in v] == gold["rng7_uniform_int_1000_1_2_3_1e9p7_5e7_100"]


def test_log_sum_exp_matches_reference(oracle, gold):
    cases = [[-1.0, -2.0, -3.0], [-1e3, -1e3 - 1e-9, -745.0, -2000.0], [-np.inf, -np.inf], [-np.inf, 0.5]]
    want = [float(x) for x in gold["log_sum_exp_abcd"]]
    for c, w in zip(cases, want):
        got = oracle.log_sum_exp(c)
        assert got == w or (np.isinf(got) and np.isinf(w) and got == w)


def test_survey_appendix_c(oracle):
    # SURVEY.md Appendix C, produced from the same compiled reference headers
    assert [oracle.uniform_component(0, 0, n, 100) for n in (0, 1, 2, 12345, 19999)] == [66, 30, 4, 13, 73]
    assert [oracle.uniform_component(0, 7, n, 50000) for n in (0, 1, 2, 12345, 49999999)] == [9107, 40268, 44727, 28456, 25456]


# ------------------------------------------------------------------ SPEC known answers
def test_spec_precompute_kat(oracle):
    # D=2, H=1, Lambda=(1,0)^T, Psi=I -> L=[2], log|Sigma|=ln 2, V=(0.5, 0)
    p = oracle.Params(np.array([1.0]), np.zeros((1, 2)), np.array([[[1.0, 0.0]]]), np.ones((1, 2)))
    k = oracle.precompute_all(p)
    assert k.Lmat[0, 0, 0] == 2.0
    assert abs(k.logdet[0] - np.log(2)) < 1e-15
    np.testing.assert_allclose(k.V[0, :, 0], [0.5, 0.0], atol=1e-16)
    # Lambda = 0 -> L = I, V = 0, log|Sigma| = sum log psi
    psi = np.array([[0.5, 2.0, 3.0]])
    p = oracle.Params(np.array([1.0]), np.zeros((1, 3)), np.zeros((1, 2, 3)), psi)
    k = oracle.precompute_all(p)
    np.testing.assert_array_equal(k.Lmat[0], np.eye(2))
    np.testing.assert_array_equal(k.V[0], 0.0)
    assert abs(k.logdet[0] - np.log(psi).sum()) < 1e-14


def test_spec_log_joint_kat(oracle):
    # standard normal at its mode
    p = oracle.Params(np.array([1.0]), np.zeros((1, 1)), np.zeros((1, 1, 1)), np.ones((1, 1)))
    k = oracle.precompute_all(p)
    assert abs(oracle.log_joint(k, p.mu, 0, np.zeros(1, np.float32)) - (-0.5 * np.log(2 * np.pi))) < 1e-14
    # SPEC.md:69 (value -3.62755 as printed; exact ln .5 - ln 2pi - .5 ln 2 - .75)
    p = oracle.Params(np.array([0.5, 0.5]), np.zeros((2, 2)), np.array([[[1.0, 0.0]]] * 2), np.ones((2, 2)))
    k = oracle.precompute_all(p)
    v = oracle.log_joint(k, p.mu, 0, np.array([1, 1], np.float32))
    exact = np.log(0.5) - np.log(2 * np.pi) - 0.5 * np.log(2) - 0.75
    assert abs(v - exact) < 1e-14 and abs(v - (-3.62755)) < 1e-4


def dense_log_joint(p, c, x):
    """proj/tests/oracle.hpp:18-37 semantics: dense Sigma, LU log-det, solve."""
    lam = p.lam[c].T  # D x H
    S = lam @ lam.T + np.diag(p.psi[c])
    v = x.astype(np.float64) - p.mu[c]
    sign, ld = np.linalg.slogdet(S)
    assert sign > 0
    return np.log(p.pi[c]) - 0.5 * (len(x) * np.log(2 * np.pi) + ld + v @ np.linalg.solve(S, v))


def test_woodbury_matches_dense_covariance(oracle):
    # acceptance criterion 1: >=1000 random (params, x), D in 2..16, H in 1..4
    rng = np.random.default_rng(0)
    worst = 0.0
    for t in range(1000):
        D = int(rng.integers(2, 17))
        H = int(rng.integers(1, min(4, D) + 1))
        p = oracle.Params(np.array([rng.uniform(0.2, 1.0)]), 3 * rng.normal(size=(1, D)),
                          rng.normal(size=(1, H, D)), rng.uniform(0.2, 2.0, (1, D)))
        k = oracle.precompute_all(p)
        x = rng.normal(size=D).astype(np.float32) * 3
        worst = max(worst, abs(oracle.log_joint(k, p.mu, 0, x) - dense_log_joint(p, 0, x)))
    assert worst < 1e-8, worst


def _estep_problem(oracle, N=400, D=6, C=12, H=2, Cp=3, G=4, seed=0):
    X, _ = gaussian_problem(N, D, 6, 2, seed=seed)
    p, st, floor, _ = oracle.initialize(X, C, H, Cp, G, seed=seed, scale=0.1, loading_init=1)
    return X, p, st, floor


def test_search_space_union_fig1(oracle):
    # K={35,87,42}, g_35={98,35,23}, g_87={16,87,63}, g_42={37,42,8};
    # extra already present -> S = {98,35,23,16,87,63,37,42,8} (insertion order of sorted rows)
    C = 100
    seed, it = 0, 0
    n_extra = None
    # find a row index whose extra draw falls inside the union
    union = {98, 35, 23, 16, 87, 63, 37, 42, 8}
    for n in range(10000):
        if oracle.uniform_component(seed, it, n, C) in union:
            n_extra = n
            break
    N = n_extra + 1
    D = 2
    X = np.zeros((N, D), np.float32)
    K = np.tile(np.array([[0, 1, 2]], np.int32), (N, 1))
    K[n_extra] = [35, 42, 87]
    g = np.full((C, 3), -1, np.int32)
    gc = np.ones(C, np.int32)
    for c in range(C):
        g[c, 0] = c
    for c, row in ((35, [23, 35, 98]), (87, [16, 63, 87]), (42, [8, 37, 42])):
        g[c] = row
        gc[c] = 3
    p = oracle.Params(np.full(C, 1.0 / C), np.zeros((C, D)), np.zeros((C, 1, D)), np.ones((C, D)))
    k = oracle.precompute_all(p)
    st = oracle.State(K, g, gc)
    e = oracle.variational_e_step(X, p, k, st, seed, it)
    S = e.idx[n_extra, :e.count[n_extra]]
    assert set(S.tolist()) == union and len(S) == 9
    # insertion order: g rows of K members in ascending K order (estep.cpp:83-101)
    assert S.tolist() == [23, 35, 98, 8, 37, 42, 16, 63, 87]


def test_update_k_and_partition_ties(oracle):
    # SPEC.md:153-155 / 163-165: top-C' by (l desc, index asc); label ties -> smaller index
    C, D = 4, 1
    N = 1
    X = np.zeros((N, D), np.float32)
    p = oracle.Params(np.full(C, 0.25), np.zeros((C, D)), np.zeros((C, 1, D)), np.ones((C, D)))
    k = oracle.precompute_all(p)  # identical components: all joints tie exactly
    g = np.array([[0, 1, 2, 3]] * C, np.int32)
    st = oracle.State(np.array([[2, 3]], np.int32), g, np.full(C, 4, np.int32))
    oracle.variational_e_step(X, p, k, st, 0, 0)
    assert st.K.tolist() == [[0, 1]]  # ties broken by the smaller index
    assert st.labels.tolist() == [0]


def test_update_g_kat(oracle):
    # keys {a:0.1, b:0.5, d:0.2}, G=3 -> g_c = {c, a, d}. Built from a
    # one-point partition whose kl values equal the targets (pi equal, l chosen).
    C, D = 4, 1
    c, a, b, d = 0, 1, 2, 3
    # l(n,ct) = l(n,c) - value  (kl mode, equal pi) -> mu offsets give the joints
    vals = {a: 0.1, b: 0.5, d: 0.2}
    mu = np.zeros((C, D))
    for ct, v in vals.items():
        mu[ct, 0] = np.sqrt(2 * v)  # -0.5 (x - mu)^2 = -v at x = 0
    p = oracle.Params(np.full(C, 0.25), mu, np.zeros((C, 1, D)), np.ones((C, D)))
    k = oracle.precompute_all(p)
    X = np.zeros((1, D), np.float32)
    g = np.array([[0, 1, 2, 3]] * C, np.int32)
    st = oracle.State(np.array([[0]], np.int32), g, np.full(C, 4, np.int32))
    st.g_count[:] = 4
    # G=3 view: rebuild with G=3 (g rows of length 3 containing all needed keys via K={0} and g_0)
    g3 = np.array([[0, 1, 2], [1, 2, 3], [0, 2, 3], [0, 1, 3]], np.int32)
    g3[0] = [0, 1, 2]
    st = oracle.State(np.array([[0]], np.int32), np.array([[0, 1, 2], [1, 2, 3], [2, 3, 0], [3, 0, 1]], np.int32),
                      np.full(C, 3, np.int32))
    st.g[2] = [0, 2, 3]
    st.g[3] = [0, 1, 3]
    st.g[0] = [0, 1, 2]
    e = oracle.variational_e_step(X, p, k, st, 0, 0, dump_distances=True)
    S = set(e.idx[0, :e.count[0]].tolist())
    dc, dct, ds, dn = e.dist
    got = {int(t): s / n for cc, t, s, n in zip(dc, dct, ds, dn) if cc == 0}
    for t in got:
        assert abs(got[t] - vals[t]) < 1e-12
    if S >= {0, 1, 2, 3}:
        assert st.g[0, :st.g_count[0]].tolist() == [0, 1, 3]  # {c, a, d}


def test_responsibilities_kat(oracle):
    # two members with equal joints -> (0.5, 0.5)
    C, D = 2, 1
    p = oracle.Params(np.full(C, 0.5), np.zeros((C, D)), np.zeros((C, 1, D)), np.ones((C, D)))
    k = oracle.precompute_all(p)
    st = oracle.State(np.array([[0, 1]], np.int32), np.array([[0, 1], [0, 1]], np.int32), np.full(C, 2, np.int32))
    e = oracle.variational_e_step(np.zeros((1, D), np.float32), p, k, st, 0, 0)
    np.testing.assert_allclose(e.resp[0], [0.5, 0.5], atol=1e-15)


def test_suffstats_zero_loading_kat(oracle):
    # Lambda=0 -> mz=0, Sigma_z=I, E_c = N_c blockdiag(I,1), Y_c = [0 | sum q x]
    X, _ = gaussian_problem(200, 5, 3, 2, seed=2)
    C, H, Cp = 3, 2, 2
    p = oracle.Params(np.full(C, 1 / 3), np.zeros((C, 5)), np.zeros((C, H, 5)), np.ones((C, 5)))
    k = oracle.precompute_all(p)
    rng = np.random.default_rng(0)
    K = np.sort(np.stack([rng.choice(C, Cp, replace=False) for _ in range(200)]), axis=1).astype(np.int32)
    q = rng.dirichlet(np.ones(Cp), 200)
    s = oracle.accumulate_suffstats(X, p, k, K, q)
    for c in range(C):
        want = np.zeros((H + 1, H + 1))
        want[:H, :H] = s.Nc[c] * np.eye(H)
        want[H, H] = s.Nc[c]
        np.testing.assert_allclose(s.E[c], want, atol=1e-12)
        np.testing.assert_allclose(s.Y[c, :H], 0.0, atol=1e-12)
        w = (q * (K == c)).sum(1)
        np.testing.assert_allclose(s.Y[c, H], (w[:, None] * X).sum(0), rtol=1e-12)


def test_update_params_c1_kat(oracle):
    # C=1, Lambda=0, q=1 -> mu = sample mean, sigma^2 = biased sample variance
    X, _ = gaussian_problem(500, 4, 2, 1, seed=4)
    p = oracle.Params(np.ones(1), np.zeros((1, 4)), np.zeros((1, 1, 4)), np.ones((1, 4)))
    k = oracle.precompute_all(p)
    K = np.zeros((500, 1), np.int32)
    s = oracle.accumulate_suffstats(X, p, k, K, np.ones((500, 1)))
    floor = np.full(4, 1e-8)
    p2 = oracle.update_params(s, 500, p, floor)
    Xd = X.astype(np.float64)
    np.testing.assert_allclose(p2.mu[0], Xd.mean(0), rtol=1e-10)
    np.testing.assert_allclose(p2.psi[0], Xd.var(0), rtol=1e-8)
    assert p2.pi[0] == 1.0


def test_no_truncation_limit_equals_exact_em(oracle):
    # acceptance criterion 2: C'=C, G=C -> F equals the exact LL
    X, _ = gaussian_problem(300, 6, 4, 2, seed=8)
    C, H = 4, 2
    p, st, floor, _ = oracle.initialize(X, C, H, C, C, seed=1, scale=0.1, loading_init=1)
    k = oracle.precompute_all(p)
    e = oracle.variational_e_step(X, p, k, st, 0, 0)
    ll = oracle.exact_log_likelihood(X, p, k)
    assert abs(e.F - ll) <= 1e-10 * abs(ll)
    for _ in range(5):
        s = oracle.accumulate_suffstats(X, p, k, st.K, e.resp)
        p = oracle.update_params(s, X.shape[0], p, floor)
        k = oracle.precompute_all(p)
        F = oracle.truncated_free_energy(X, p, k, st.K)
        assert abs(F - oracle.exact_log_likelihood(X, p, k)) <= 1e-10 * abs(F)
        e = oracle.variational_e_step(X, p, k, st, 0, 1)


def test_monotone_free_energy_and_joint_bound(oracle):
    # acceptance criteria 3 and 6
    for seed in range(6):
        X, p, st, floor = _estep_problem(oracle, N=300, D=5, C=10, H=2, Cp=2, G=3, seed=seed)
        k = oracle.precompute_all(p)
        F_prev = oracle.truncated_free_energy(X, p, k, st.K)
        for it in range(4):
            e = oracle.variational_e_step(X, p, k, st, seed, it)
            assert e.F >= F_prev - 1e-9 * abs(F_prev)
            assert e.joints <= X.shape[0] * (2 * 3 + 1)
            s = oracle.accumulate_suffstats(X, p, k, st.K, e.resp)
            p = oracle.update_params(s, X.shape[0], p, floor)
            k = oracle.precompute_all(p)
            F_prev = oracle.truncated_free_energy(X, p, k, st.K)
            assert F_prev >= e.F - 1e-9 * abs(e.F)


def test_thread_count_invariance(oracle):
    # acceptance criterion 12 + SURVEY App. E.11: integer state independent of threads
    X, p, st, floor = _estep_problem(oracle, N=2000, D=8, C=30, H=2, Cp=3, G=5, seed=3)
    k = oracle.precompute_all(p)
    a, b = st.copy(), st.copy()
    ea = oracle.variational_e_step(X, p, k, a, 0, 0, threads=1)
    eb = oracle.variational_e_step(X, p, k, b, 0, 0, threads=7)
    assert np.array_equal(a.K, b.K) and np.array_equal(a.g, b.g) and ea.joints == eb.joints
    assert abs(ea.F - eb.F) <= 1e-12 * abs(ea.F)


def test_sharded_extra_draws_use_global_index(oracle):
    X, p, st, floor = _estep_problem(oracle, N=600, D=4, C=20, H=1, Cp=2, G=3, seed=5)
    k = oracle.precompute_all(p)
    full = st.copy()
    e = oracle.variational_e_step(X, p, k, full, 9, 4)
    part = oracle.State(st.K[300:].copy(), st.g.copy(), st.g_count.copy())
    e2 = oracle.variational_e_step(X[300:], p, k, part, 9, 4, n_offset=300)
    assert np.array_equal(e2.idx, e.idx[300:])
    assert np.array_equal(part.K, full.K[300:])


def test_update_params_ldlt_semantics(oracle):
    # mstep.cpp:129-140 factorises E_c with Eigen LDLT: singular/indefinite E_c
    # solve through the pivoted LDL^T and D's pseudo-inverse; a zero pivot
    # followed by a non-zero one takes the jitter retry
    from _helpers import ldlt_cases
    s, prev, floor, want = ldlt_cases(oracle)
    p = oracle.update_params(s, 10, prev, floor)
    H = prev.H
    for c in range(4):
        # c2's jittered E has condition ~1.5e10: fp64 solves agree to ~cond*eps
        tol = dict(rtol=0, atol=2e-5) if c == 2 else dict(rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(p.lam[c], want[c, :H], err_msg=str(c), **tol)
        np.testing.assert_allclose(p.mu[c], want[c, H], err_msg=str(c), **tol)
    # a solution that overflows with and without the jitter -> SingularEc
    s.E[3] = np.diag([1e-300, 1e-300, 1e-300])
    s.Nc[3] = 1e-300
    s.Y[3] = 1e10
    with pytest.raises(oracle.OracleError, match="component 3"):
        oracle.update_params(s, 10, prev, floor)


def test_em_full_step_is_the_no_truncation_limit(oracle):
    """em_full_step's log-likelihood is exact_log_likelihood, its responsibilities
    sum to 1 per point, and with C' = C (no truncation) the
    variational E-step's statistics equal em_full_step's."""
    O = oracle
    from _helpers import gaussian_problem
    X, _ = gaussian_problem(600, 12, 5, 2, seed=8)
    C, H = 6, 2
    p, st, floor, _ = O.initialize(X, C, H, C, C, seed=0, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    s_em, ll, joints = O.em_full_step(X, p, k, threads=2)
    assert joints == X.shape[0] * C
    assert abs(ll - O.exact_log_likelihood(X, p, k)) <= 1e-10 * abs(ll)
    np.testing.assert_allclose(s_em.Nc.sum(), X.shape[0], rtol=1e-12)
    e = O.variational_e_step(X, p, k, st, 0, 0, threads=2)
    assert abs(e.F - ll) <= 1e-10 * abs(ll)
    s_v = O.accumulate_suffstats(X, p, k, st.K, e.resp, threads=2)
    for f in ("Nc", "E", "Y", "sq"):
        np.testing.assert_allclose(getattr(s_v, f), getattr(s_em, f), rtol=1e-10, atol=1e-10, err_msg=f)


def test_afkmc2_oracle_properties(oracle):
    """afkmc2_seed restatement: the first seed is the stream's first
    uniform_int(N) (seeding.cpp:70), seeds are distinct rows, chain_length = 1
    makes every later seed the first cdf draw, and the squared-distance count
    is N + m * sum_{k<C} k (seeding.cpp:77-101, no fallback)."""
    O = oracle
    from _helpers import gaussian_problem
    X, _ = gaussian_problem(800, 6, 4, 2, seed=9)
    seed = O.hash_combine(1, O.INIT_SALT)
    C, m = 15, 4
    s, st, n = O.afkmc2_seed(X, C, m, seed)
    first = O.rng_ops(seed, [2], [X.shape[0]])  # op 2: uniform_int(bound)
    assert s[0] == int(first[0])
    assert len(set(s.tolist())) == C
    assert n == X.shape[0] + m * sum(range(1, C))
