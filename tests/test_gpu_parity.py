"""GPU parity: the CUDA path through the C-ABI vs the fp64 oracle on the same
seeded inputs (teacher-forced per step, then free-running), SURVEY §4/§8(c)."""
import numpy as np
import pytest

from _helpers import (LJ_RTOL, compare_estep, compare_g, gaussian_problem, to_oracle_params,
                      to_oracle_state, to_vmfa_params, to_vmfa_state)

pytestmark = pytest.mark.gpu


def _setup(O, V, X, C, H, Cp, G, seed=0, loading_init=1, scale=0.1):
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=seed, scale=scale, loading_init=loading_init)
    sess = V.Session(C, X.shape[1], H, Cp, G, X)
    sess.set_floor(floor)
    sess.upload_params(to_vmfa_params(V, p))
    sess.upload_state(to_vmfa_state(V, st))
    return p, st, floor, sess


def _estep_both(O, V, sess, X, p, st, seed, it, mode=0, dump=True):
    k = O.precompute_all(p)
    st_or = st.copy()
    e_or = O.variational_e_step(X, p, k, st_or, seed, it, mode=mode, threads=4, dump_distances=dump)
    if dump:
        sess.arm_distance_dump()
    sess.upload_state(to_vmfa_state(V, st))
    F, J = sess.variational_e_step(seed, it, mode)
    ret = sess.download_estep()
    st_g = sess.download_state()
    return e_or, st_or, F, J, ret, st_g, k


def test_precompute_caches_match_oracle(oracle, gpu):
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 24, 12, 3, seed=1)
    for H in (1, 3, 4, 8, 16):
        p, st, floor, sess = _setup(O, V, X, 12, H, 2, 4)
        p.lam[:] = np.random.default_rng(H).normal(0, 0.7, p.lam.shape)
        p.psi[:] = np.random.default_rng(H + 1).uniform(0.05, 2.0, p.psi.shape)
        p.pi[:] = np.random.default_rng(H + 2).dirichlet(np.ones(12))
        p.pi[3] = 0.0
        p.pi /= p.pi.sum()
        sess.upload_params(to_vmfa_params(V, p))
        k = O.precompute_all(p)
        got = sess.download_caches()
        for name in ("U", "Lmat", "V", "Sz", "inv_psi", "logdet"):
            ref = getattr(k, name)
            np.testing.assert_allclose(got[name], ref, rtol=1e-10, atol=1e-12, err_msg=name)
        assert got["log_pi"][3] == -np.inf
        np.testing.assert_allclose(got["log_pi"][np.isfinite(k.log_pi)], k.log_pi[np.isfinite(k.log_pi)], rtol=1e-14)
        sess.close()


@pytest.mark.parametrize("case", [
    dict(N=4000, D=64, C=100, H=4, Cp=3, G=5),    # config 1 shape
    dict(N=4000, D=256, C=200, H=8, Cp=5, G=10),  # config 2 shape
    dict(N=1500, D=32, C=12, H=2, Cp=3, G=5),     # C < C'G+1: stride = C
    dict(N=2000, D=16, C=40, H=1, Cp=1, G=1),     # C'=1, G=1
    dict(N=1000, D=10, C=6, H=2, Cp=6, G=6),      # C'=C: no truncation
    dict(N=2000, D=100, C=50, H=16, Cp=4, G=8),   # H=16 chunk
    dict(N=1500, D=64, C=60, H=12, Cp=3, G=18),   # two component groups per anchor job (G > 15)
])
@pytest.mark.parametrize("scorer", ["ws", "ws-imagefree", "ws-imagefree-only", "tc", "ffma"])
def test_estep_teacher_forced(oracle, gpu, case, scorer, monkeypatch):
    # ws-imagefree: the warp-specialised scorer assembling each anchor stage
    # from the one-component images (VMFA_IMAGE_FREE=1, opt-in); -only: the
    # route without any full anchor images (VMFA_IMAGE_FREE=2, config 5)
    O, V = oracle, gpu
    monkeypatch.setenv("VMFA_SCORER", scorer.split("-")[0])
    if scorer == "ws-imagefree":
        monkeypatch.setenv("VMFA_IMAGE_FREE", "1")
    if scorer == "ws-imagefree-only":
        monkeypatch.setenv("VMFA_IMAGE_FREE", "2")
    X, _ = gaussian_problem(case["N"], case["D"], max(case["C"] // 2, 2), min(case["H"], 4), seed=7)
    C, H, Cp, G = case["C"], case["H"], case["Cp"], case["G"]
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    rep = {}
    for it in range(3):  # teacher-forced consecutive E-steps (warm-up style)
        e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 11, it)
        compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp, rep)
        same_part = np.ones(C, bool)
        diff_rows = np.any(st_g.K != st_or.K, axis=1) | (st_g.labels != st_or.labels)
        for n in np.nonzero(diff_rows)[0]:
            same_part[st_or.labels[n]] = False
            same_part[st_g.labels[n]] = False
        bad = compare_g(st_g.g, st_g.g_count, st_or.g, st_or.g_count, e_or.dist, same_part)
        assert not bad, f"g differs outside near-ties for components {bad[:10]}"
        # block-3 accumulators: exact counts, sums within the log-joint tolerance
        dc, dct, ds, dn = sess.download_distances()
        oc, oct_, os_, on = e_or.dist
        if not diff_rows.any():
            assert np.array_equal(dc, oc) and np.array_equal(dct, oct_) and np.array_equal(dn, on)
            np.testing.assert_allclose(ds, os_, rtol=1e-4, atol=1e-3 * np.abs(os_).max())
        st = st_or  # teacher forcing: continue from the oracle's state
    sess.close()


@pytest.mark.parametrize("scorer", ["ws", "tc"])
def test_estep_config3_shape(oracle, gpu, scorer, monkeypatch):
    # BASELINE config 3's shape (D = 784, H = 16, C' = 5, G = 10) at a small N
    # (the FFMA cross-check scorer's tile stops at D = 775)
    O, V = oracle, gpu
    monkeypatch.setenv("VMFA_SCORER", scorer)
    X, _ = gaussian_problem(1500, 784, 20, 4, seed=13)
    C, H, Cp, G = 40, 16, 5, 10
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    for it in range(2):
        e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 3, it)
        compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
        st = st_or
    sess.close()


def test_estep_large_C_dense_rows(oracle, gpu):
    # C - 1 > kGupdCap / 2: every block-3 item adds its exact partial table into
    # the dense rows through a small hash (overflowing keys go straight to the
    # rows), selection from the rows for all components
    O, V = oracle, gpu
    X, _ = gaussian_problem(24000, 8, 3000, 2, seed=17)
    C, H, Cp, G = 4500, 2, 3, 5
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    for it in range(2):
        e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 5, it)
        compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
        same_part = np.ones(C, bool)
        diff_rows = np.any(st_g.K != st_or.K, axis=1) | (st_g.labels != st_or.labels)
        for n in np.nonzero(diff_rows)[0]:
            same_part[st_or.labels[n]] = False
            same_part[st_g.labels[n]] = False
        bad = compare_g(st_g.g, st_g.g_count, st_or.g, st_or.g_count, e_or.dist, same_part)
        assert not bad, f"g differs outside near-ties for components {bad[:10]}"
        st = st_or
    sess.close()


def test_estep_euclid_and_frozen(oracle, gpu):
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 48, 30, 3, seed=3)
    C, H, Cp, G = 60, 3, 3, 6
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    p.pi[[1, 5, 9]] = 0.0  # frozen empty components: -inf joints, still counted
    p.pi /= p.pi.sum()
    sess.upload_params(to_vmfa_params(V, p))
    for mode in (1, 0):
        e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 5, 2, mode=mode)
        compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
        # block 3 skips frozen candidates (pi = 0, estep.cpp:301): a frozen
        # component appears in no neighbourhood but its own
        for c in range(C):
            others = [v for v in st_g.g[c, :st_g.g_count[c]] if v != c]
            assert not np.isin(others, [1, 5, 9]).any(), (c, others)
    sess.close()


def test_block3_values_beyond_2_31_match_oracle(oracle, gpu):
    """Block-3 values far beyond 2^31 (components with Psi at a tiny floor:
    v^2/psi ~ 1e9 per dimension) are summed exactly by the fixed-point
    accumulator (range 2^40) and agree with the oracle's fp64 sums."""
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 32, 12, 2, seed=23)
    C, H, Cp, G = 24, 2, 3, 5
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    p.psi[[2, 7, 11]] = 1e-8
    sess.upload_params(to_vmfa_params(V, p))
    e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 4, 1)
    compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
    dc, dct, ds, dn = sess.download_distances()
    oc, oct_, os_, on = e_or.dist
    assert np.abs(os_).max() > 2.0 ** 31 * 10  # the sums really exceed the old saturation bound
    diff_rows = np.any(st_g.K != st_or.K, axis=1) | (st_g.labels != st_or.labels)
    assert not diff_rows.any()
    assert np.array_equal(dc, oc) and np.array_equal(dct, oct_) and np.array_equal(dn, on)
    np.testing.assert_allclose(ds, os_, rtol=1e-5)
    assert np.array_equal(st_g.g, st_or.g)
    sess.close()


@pytest.mark.parametrize("case", [
    dict(N=5000, D=40, C=30, H=3, Cp=3, G=5),     # 5-column statistics pass
    dict(N=4000, D=256, C=60, H=8, Cp=5, G=10),   # config 2 shape: 9-column pass, bulk row gather
    dict(N=3000, D=30, C=25, H=16, Cp=3, G=5),    # 17-column pass, D % 4 != 0 (4-byte gather)
    dict(N=2500, D=64, C=20, H=20, Cp=3, G=4),    # H + 1 > 17: two column passes + separate E pass
    dict(N=1500, D=784, C=24, H=16, Cp=5, G=10),  # config 3 shape (D = 784)
    dict(N=4000, D=64, C=40, H=4, Cp=3, G=5),     # config 1 shape (tensor-core pass: 1 dim tile per warp)
    dict(N=3000, D=256, C=30, H=15, Cp=3, G=5),   # H + 1 = 16: two latent n-tiles, full m16 tile
    dict(N=3000, D=512, C=30, H=8, Cp=3, G=5),    # 8 dimension tiles per warp
    dict(N=3000, D=48, C=30, H=10, Cp=3, G=5),    # D/8 = 6 tiles < 8 warps, XS % 32 != 4
    dict(N=3000, D=64, C=30, H=16, Cp=3, G=5),    # H + 1 = 17: constant column by FFMA (16-row batches)
    dict(N=2000, D=1000, C=16, H=6, Cp=3, G=5),   # 16 dimension tiles per warp (D > 832)
])
@pytest.mark.parametrize("stats", ["tc", "mma", "ffma"])
def test_mstep_parity(oracle, gpu, case, stats, monkeypatch):
    # mma: the default mma.sync kernel (FFMA beyond its shapes); tc: the
    # tcgen05 kernel (opt-in, H <= 16, D <= 832); ffma: the FFMA cross-check
    O, V = oracle, gpu
    if stats == "mma":
        monkeypatch.delenv("VMFA_STATS", raising=False)
    else:
        monkeypatch.setenv("VMFA_STATS", stats)
    X, _ = gaussian_problem(case["N"], case["D"], max(4, case["C"] // 2), min(case["H"], 4), seed=5)
    C, H, Cp, G = case["C"], case["H"], case["Cp"], case["G"]
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    sess.variational_e_step(0, 0)
    _, _, _, resp = sess.download_estep()
    st_g = sess.download_state()
    k = O.precompute_all(p)
    s_or = O.accumulate_suffstats(X, p, k, st_g.K, resp, threads=4)
    sess.accumulate_suffstats()
    s_g = sess.download_suffstats()
    # N_c: fp32 tile sums of q / q_max, rescaled in fp64 (exactly 0 iff every q is 0)
    np.testing.assert_allclose(s_g.Nc, s_or.Nc, rtol=1e-6, atol=0)
    assert np.array_equal(s_g.Nc == 0.0, s_or.Nc == 0.0)
    if stats == "tc":
        # 3xFP16 with fp32 TMEM accumulation over up to 52 k-steps: ~5e-6 of
        # each component's largest entry (tests/test_gpu_parity_scale.py's measure)
        for f in ("E", "Y", "sq"):
            a, b = getattr(s_g, f).reshape(C, -1), getattr(s_or, f).reshape(C, -1)
            rel = np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-300)
            assert rel.max() <= 2e-5, (f, float(rel.max()))
    else:
        np.testing.assert_allclose(s_g.E, s_or.E, rtol=1e-5, atol=1e-6 * np.abs(s_or.E).max())
        np.testing.assert_allclose(s_g.Y, s_or.Y, rtol=1e-5, atol=1e-6 * np.abs(s_or.Y).max())
        # centred fp32 accumulation restored in fp64: ~1e-6 relative
        np.testing.assert_allclose(s_g.sq, s_or.sq, rtol=1e-5)
    # update_params from identical statistics: fp64 on both sides
    sess.upload_suffstats(s_or)
    sess.update_params()
    p_g = sess.download_params()
    p_or = O.update_params(s_or, X.shape[0], p, floor)
    for f in ("pi", "mu", "lam", "psi"):
        np.testing.assert_allclose(getattr(p_g, f), getattr(p_or, f), rtol=1e-9, atol=1e-12, err_msg=f)
    # post-M-step truncated free energy with the new caches
    F_g = sess.truncated_free_energy()
    F_or = O.truncated_free_energy(X, p_or, O.precompute_all(p_or), st_g.K, threads=4)
    assert abs(F_g - F_or) <= 1e-5 * abs(F_or)
    sess.close()


def test_update_freezes_empty_component(oracle, gpu):
    O, V = oracle, gpu
    X, _ = gaussian_problem(2000, 12, 8, 2, seed=9)
    C, H, Cp, G = 10, 2, 2, 3
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    sess.variational_e_step(0, 0)
    sess.accumulate_suffstats()
    s = sess.download_suffstats()
    s.Nc[4] = 0.0
    s.Y[4] = 0
    s.E[4] = 0
    s.sq[4] = 0
    sess.upload_suffstats(s)
    sess.update_params()
    p_g = sess.download_params()
    p_or = O.update_params(s, X.shape[0], p, floor)
    assert p_g.pi[4] == 0.0 and p_or.pi[4] == 0.0
    np.testing.assert_array_equal(p_g.mu[4], p.mu[4])
    np.testing.assert_array_equal(p_g.lam[4], p.lam[4])
    np.testing.assert_allclose(p_g.pi, p_or.pi, rtol=1e-12)
    sess.close()


def test_update_ldlt_semantics_match_oracle(oracle, gpu):
    # singular / indefinite / jitter-path E_c (mstep.cpp:129-140): the device
    # LDLT restatement and the oracle's agree; an overflowing solve -> SingularEc
    from _helpers import ldlt_cases
    O, V = oracle, gpu
    s, prev, floor, want = ldlt_cases(O)
    X = np.random.default_rng(2).normal(size=(10, 5)).astype(np.float32)
    sess = V.Session(4, 5, 2, 2, 2, X)
    sess.set_floor(floor)
    sess.upload_params(to_vmfa_params(V, prev))
    sess.upload_suffstats(s)
    sess.update_params()
    p_g = sess.download_params()
    p_or = O.update_params(s, 10, prev, floor)
    for f in ("pi", "mu", "psi"):
        np.testing.assert_allclose(getattr(p_g, f), getattr(p_or, f), rtol=1e-12, atol=1e-14, err_msg=f)
    for c in (0, 1, 3):
        np.testing.assert_allclose(p_g.lam[c], p_or.lam[c], rtol=1e-12, atol=1e-14, err_msg=f"lam[{c}]")
    # c2 is solved through the jitter retry: E_2 + 1e-10 tr/H1 I has condition
    # number ~1.5e10, so any two fp64 LDLTs differ by ~cond * eps * |Y| ~ 1e-5
    np.testing.assert_allclose(p_g.lam[2], p_or.lam[2], rtol=0, atol=2e-5, err_msg="lam[2]")
    np.testing.assert_allclose(p_g.lam[1], want[1, :2], rtol=1e-12, atol=1e-14)
    s.E[3] = np.diag([1e-300, 1e-300, 1e-300])
    s.Nc[3] = 1e-300
    s.Y[3] = 1e10
    sess.upload_params(to_vmfa_params(V, prev))
    sess.upload_suffstats(s)
    with pytest.raises(V.VmfaError, match="SingularEc"):
        sess.update_params()
    sess.close()


def test_free_running_config1(oracle, gpu):
    """Config 1 (BASELINE.json configs[0]) end to end: 2 warm-up E-steps + 20
    iterations from the same seeded init; F per iteration within 1e-4 relative,
    joint counts and final parameters compared."""
    O, V = oracle, gpu
    X = V.gen_synthetic(V.synth_spec(1))
    cfg = V.CONFIGS[1]["model"]
    C, H, Cp, G = cfg["C"], cfg["H"], cfg["Cp"] if "Cp" in cfg else cfg["Cprime"], cfg["G"]
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    recs_g = V.train_fixed(sess, 0, 2, 20)
    p_or, st_or, recs_o = O.train_fixed(X, p.copy(), st.copy(), floor, 0, 2, 20, threads=8)
    for rg, ro in zip(recs_g, recs_o):
        assert abs(rg["F"] - ro["F"]) <= LJ_RTOL * abs(ro["F"]), (rg, ro)
    Jg = sum(r["joints"] for r in recs_g)
    Jo = sum(r["joints"] for r in recs_o)
    assert abs(Jg - Jo) <= 1e-3 * Jo
    # final parameters after the fixed 2 + 20 iterations, free-running: the
    # trajectories share every decision except near-ties, so
    # the parameters agree to the tolerances below, relative to each
    # component's largest magnitude of that parameter (measured on B200: see
    # DESIGN.md §5 and $PARITY_REPORT_DIR/parity_config1_free.json)
    p_g = sess.download_params()
    tols = {"pi": (1e-2, 1e-4), "mu": (1e-2, 1e-4), "lam": (5e-2, 1e-3), "psi": (1e-2, 1e-4)}  # (max, median)
    rep = {}
    for f in tols:
        a, b = getattr(p_g, f), getattr(p_or, f)
        a2, b2 = a.reshape(C, -1), b.reshape(C, -1)
        rel = np.abs(a2 - b2).max(axis=1) / np.maximum(np.abs(b2).max(axis=1), 1e-300)
        rep[f] = dict(max=float(rel.max()), q99=float(np.quantile(rel, 0.99)), median=float(np.median(rel)))
    rep["F_rel_max"] = max(abs(rg["F"] - ro["F"]) / abs(ro["F"]) for rg, ro in zip(recs_g, recs_o))
    rep["K_rows_identical"] = float(np.mean(np.all(sess.download_state().K == st_or.K, axis=1)))
    import json
    import os
    if os.environ.get("PARITY_REPORT_DIR"):
        os.makedirs(os.environ["PARITY_REPORT_DIR"], exist_ok=True)
        with open(os.path.join(os.environ["PARITY_REPORT_DIR"], "parity_config1_free.json"), "w") as fh:
            json.dump(rep, fh, indent=1)
    for f, (tmax, tmed) in tols.items():
        assert rep[f]["max"] <= tmax and rep[f]["median"] <= tmed, (f, rep[f])
    sess.close()


def test_multishard_matches_single(gpu, oracle):
    """Two contexts on one GPU holding halves of the rows, combined through the
    phase API exchange buffers (summed here with torch, as NCCL would), must
    reproduce the single-context iteration: identical K, g and joint counts;
    F and parameters equal to rounding."""
    import torch
    O, V = oracle, gpu
    X, _ = gaussian_problem(6000, 32, 20, 3, seed=21)
    C, H, Cp, G = 40, 3, 3, 5
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
    single = V.Session(C, 32, H, Cp, G, X)
    single.set_floor(floor)
    single.upload_params(to_vmfa_params(V, p))
    single.upload_state(to_vmfa_state(V, st))
    half = X.shape[0] // 2
    shards = []
    for r, (a, b) in enumerate([(0, half), (half, X.shape[0])]):
        s = V.Session(C, 32, H, Cp, G, X[a:b], n_offset=a, n_total=X.shape[0])
        s.set_floor(floor)
        s.upload_params(to_vmfa_params(V, p))
        sub = V.State(st.K[a:b].copy(), st.g.copy(), st.g_count.copy())
        s.upload_state(sub)
        shards.append(s)

    class _View:
        def __init__(self, ptr, n, dt):
            self.__cuda_array_interface__ = dict(shape=(n,), typestr="<i8" if dt == 0 else "<f8",
                                                 data=(ptr, False), version=3)

    def allreduce(which):
        views = [torch.as_tensor(_View(*s.exchange_buffer(which)), device="cuda") for s in shards]
        tot = views[0] + views[1]
        for v in views:
            v.copy_(tot)
        torch.cuda.synchronize()

    for it in range(3):
        rep = single.iterate(3, it)
        for s in shards:
            s.phase_estep_local(3, it)
        allreduce(0)
        for s in shards:
            s.phase_estep_finish()
            s.phase_stats_local()
        allreduce(1)
        for s in shards:
            s.phase_update()
            s.phase_free_energy_local()
        allreduce(2)
        Fe, J, F = shards[0].phase_scalars()
        assert J == rep["joints"]
        # statistics are fp32 partials (centred) summed per shard: rounding-level differences
        assert abs(F - rep["F"]) <= 1e-7 * abs(rep["F"])
        st1 = single.download_state()
        sa, sb = shards[0].download_state(), shards[1].download_state()
        assert np.array_equal(np.concatenate([sa.K, sb.K]), st1.K)
        assert np.array_equal(sa.g, st1.g) and np.array_equal(sb.g, st1.g)
        pa, p1 = shards[0].download_params(), single.download_params()
        np.testing.assert_allclose(pa.mu, p1.mu, rtol=1e-5, atol=1e-5 * np.abs(p1.mu).max())
    for s in shards + [single]:
        s.close()


def test_cpp_mirror_matches_python_path(gpu, tmp_path):
    """The C++ drop-in (include/vmfa_b200.hpp) and the Python mirror drive the
    same C-ABI: identical trajectories (the device path is deterministic)."""
    import subprocess
    from test_abi_host import build_facade
    V = gpu
    exe = build_facade(tmp_path)
    out = subprocess.run([str(exe), "20000"], capture_output=True, text=True, check=True).stdout
    rows = [l.split() for l in out.strip().splitlines()]
    X = V.gen_synthetic(V.synth_spec(1))
    p, st, floor, _ = V.initialize(X, 100, 4, 3, 5, seed=0, scale=0.1, loading_init=1)
    s = V.Session(100, 64, 4, 3, 5, X)
    s.set_floor(floor)
    s.upload_params(p)
    s.upload_state(st)
    recs = V.train_fixed(s, 0, 2, 20)
    assert len(rows) == len(recs)
    for r, q in zip(rows, recs):
        assert float(r[1]) == pytest.approx(q["F"], rel=1e-12, abs=0)
    s.close()
    # train_vmfa (convergence-gated loop) through both mirrors
    out = subprocess.run([str(exe), "20000", "converge"], capture_output=True, text=True, check=True).stdout
    lines = out.strip().splitlines()
    fin = lines[-1].split()
    rows = [l.split() for l in lines[:-1]]
    s = V.Session(100, 64, 4, 3, 5, X)
    s.set_floor(floor)
    s.upload_params(p)
    s.upload_state(st)
    rep = V.train_vmfa(s, V.TrainConfig(epsilon=1e-4, max_iters=60, eval_nll_every=5, warmup_epsilon=1e-3,
                                        halt_on_max_iters=False))
    s.close()
    assert len(rows) == len(rep["iterations"])
    for r, q in zip(rows, rep["iterations"]):
        assert float(r[1]) == pytest.approx(q["F"], rel=1e-12, abs=0)
        if not q["warmup"] and q["t"] % 5 == 0:
            assert float(r[2]) == pytest.approx(q["nll_train"], rel=1e-12)
    assert int(fin[1]) == int(rep["converged"]) and int(fin[2]) == rep["main_iterations"]
    assert float(fin[3]) == pytest.approx(rep["nll_train"], rel=1e-12)


@pytest.mark.parametrize("scorer", ["ws", "tc"])
def test_lookahead_free_energy_is_exact(oracle, gpu, scorer, monkeypatch):
    # the truncated F read from the next E-step's anchor pass (self slots)
    # equals the one-component pass bit for bit, and the trajectory is unchanged
    O, V = oracle, gpu
    monkeypatch.setenv("VMFA_SCORER", scorer)
    X, _ = gaussian_problem(6000, 48, 24, 3, seed=21)
    C, H, Cp, G = 40, 3, 3, 6
    runs = {}
    for la in ("1", "0"):
        monkeypatch.setenv("VMFA_LOOKAHEAD", la)
        p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
        sess.variational_e_step(0, 0)
        F = []
        for it in range(1, 5):
            r = sess.iterate(0, it)
            F.append((r["F"], r["F_estep"], r["joints"]))
            if it == 2:  # an explicit truncated_free_energy call (own pass) agrees too
                assert sess.truncated_free_energy() == r["F"]
        runs[la] = (F, sess.download_state(), sess.download_params())
        sess.close()
    (F1, s1, p1), (F0, s0, p0) = runs["1"], runs["0"]
    assert F1 == F0
    assert np.array_equal(s1.K, s0.K) and np.array_equal(s1.g, s0.g)
    for f in ("pi", "mu", "lam", "psi"):
        assert np.array_equal(getattr(p1, f), getattr(p0, f)), f


@pytest.mark.parametrize("case", [dict(N=3000, D=64, C=57, H=4, G=5, frozen=()),
                                  dict(N=2500, D=100, C=40, H=8, G=10, frozen=(3, 17)),
                                  dict(N=700, D=30, C=23, H=3, G=23, frozen=(0,))])
@pytest.mark.parametrize("imagefree", ["0", "2"])
def test_exact_log_likelihood_matches_oracle(oracle, gpu, case, imagefree, monkeypatch):
    # exact_log_likelihood (model.cpp:139-148): all-pairs N x C log-joints and
    # the per-row LSE; C not a multiple of G (short last block), D % 4 != 0 and
    # frozen components (pi = 0 -> l = -inf) included; calling it leaves the
    # lookahead state of the training loop intact. imagefree "2": the route
    # taken when the full anchor images exceed the budget (config 5), where
    # every anchor stage -- the dense pass's too -- is assembled by the loader
    if imagefree != "0":
        monkeypatch.setenv("VMFA_IMAGE_FREE", imagefree)
    O, V = oracle, gpu
    X, _ = gaussian_problem(case["N"], case["D"], max(4, case["C"] // 2), 3, seed=5)
    C, H, G = case["C"], case["H"], case["G"]
    p, st, floor, sess = _setup(O, V, X, C, H, 2, G)
    sess.variational_e_step(0, 0)
    r1 = sess.iterate(0, 1)
    pc = sess.download_params()
    if case["frozen"]:
        pi = pc.pi.copy()
        pi[list(case["frozen"])] = 0.0
        pi /= pi.sum()
        pc = V.Params(pi, pc.mu, pc.lam, pc.psi)
        sess.upload_params(pc)
    ll = sess.exact_log_likelihood()
    po = to_oracle_params(O, pc)
    ll_or = O.exact_log_likelihood(X, po, O.precompute_all(po), threads=4)
    assert np.isfinite(ll) and abs(ll - ll_or) <= 1e-5 * abs(ll_or), (ll, ll_or)
    print("exact LL rel err", abs(ll - ll_or) / abs(ll_or))
    assert sess.exact_log_likelihood() == ll  # deterministic
    if not case["frozen"]:  # the next iteration is unaffected by the dense pass
        r2 = sess.iterate(0, 2)
        p2, st2, _, s2 = _setup(O, V, X, C, H, 2, G)
        s2.variational_e_step(0, 0)
        assert s2.iterate(0, 1)["F"] == r1["F"]
        assert s2.iterate(0, 2)["F"] == r2["F"]
        s2.close()
    sess.close()


def test_no_truncation_limit_device(oracle, gpu):
    # acceptance criterion 2 on the device: C' = C, G = C ->
    # the truncated F after each M-step equals exact_log_likelihood, and both
    # match the oracle's exact LL of the same parameters. The two device passes
    # differ in centring (F: each row on its own component's mean; the dense
    # pass: on its block's first component), so they agree to the split-fp16
    # rounding of the larger centred values (measured <= 3.3e-6 relative)
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 32, 8, 2, seed=9)
    C, H = 8, 2
    p, st, floor, sess = _setup(O, V, X, C, H, C, C)
    sess.variational_e_step(0, 0)
    for it in range(1, 5):
        r = sess.iterate(0, it)
        ll = sess.exact_log_likelihood()
        assert abs(r["F"] - ll) <= 1e-5 * abs(ll), (it, r["F"], ll)
        po = to_oracle_params(O, sess.download_params())
        ll_or = O.exact_log_likelihood(X, po, O.precompute_all(po), threads=4)
        print("it", it, "F vs oracle LL", abs(r["F"] - ll_or) / abs(ll_or), "dense LL vs oracle", abs(ll - ll_or) / abs(ll_or))
        assert abs(ll - ll_or) <= 1e-5 * abs(ll_or) and abs(r["F"] - ll_or) <= 1e-5 * abs(ll_or)
    sess.close()


def test_train_vmfa_convergence_loop(oracle, gpu):
    # train_vmfa's loop (trainer.cpp:111-186): warm-up until check_convergence
    # (warmup_epsilon), main iterations until check_convergence (epsilon), NLL
    # every eval_nll_every iterations and at the end; the F sequence is the
    # fixed-count loop's, and the stop points follow the rule on it
    O, V = oracle, gpu
    X, _ = gaussian_problem(4000, 32, 12, 2, seed=4)
    C, H, Cp, G = 16, 2, 3, 4
    cfg = V.TrainConfig(seed=3, epsilon=1e-3, max_iters=200, eval_nll_every=5, warmup_epsilon=1e-3,
                        halt_on_max_iters=False)
    _, _, _, sess = _setup(O, V, X, C, H, Cp, G)
    rep = V.train_vmfa(sess, cfg)
    sess.close()
    assert rep["converged"]
    _, _, _, s2 = _setup(O, V, X, C, H, Cp, G)
    fixed = V.train_fixed(s2, 3, rep["warmup_iterations"], rep["main_iterations"])
    s2.close()
    Fw = [r["F"] for r in fixed if r["warmup"]]
    Fm = [r["F"] for r in fixed if not r["warmup"]]
    assert [r["F"] for r in rep["iterations"]] == Fw + Fm
    # warm-up stopped at the first converged step (or ran to the cap)
    stops = [i for i in range(1, len(Fw)) if V.check_convergence(Fw[i - 1], Fw[i], cfg.warmup_epsilon)]
    assert stops == [len(Fw) - 1]
    if rep["converged"]:
        stops = [i for i in range(1, len(Fm)) if V.check_convergence(Fm[i - 1], Fm[i], cfg.epsilon)]
        assert stops == [len(Fm) - 1]
    nll_recs = [r for r in rep["iterations"] if not r["warmup"] and r["t"] % 5 == 0]
    assert nll_recs and all(np.isfinite(r["nll_train"]) for r in nll_recs)
    assert rep["nll_train"] > 0 and np.isfinite(rep["nll_train"])
    # halt_on_max_iters: MaxIterExceeded at the cap
    _, _, _, s3 = _setup(O, V, X, C, H, Cp, G)
    with pytest.raises(V.VmfaError, match="MaxIterExceeded"):
        V.train_vmfa(s3, V.TrainConfig(seed=3, epsilon=1e-12, max_iters=3, warmup_epsilon=1e-3))
    s3.close()


def test_checkpoint_resume_is_exact(oracle, gpu, tmp_path):
    # MFAD + MFAM + MFAK: stop after 3 iterations, write
    # the containers, resume in a fresh session from the files -> the same
    # trajectory as the uninterrupted run, bit for bit
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 40, 10, 2, seed=6)
    C, H, Cp, G = 14, 2, 3, 4
    V.save_dataset(tmp_path / "x.mfad", X)
    p, st, floor, a = _setup(O, V, X, C, H, Cp, G)
    a.variational_e_step(0, 0)
    full = [a.iterate(0, it)["F"] for it in range(1, 7)]
    a.close()
    _, _, _, b = _setup(O, V, X, C, H, Cp, G)
    b.variational_e_step(0, 0)
    first = [b.iterate(0, it)["F"] for it in range(1, 4)]
    V.save_checkpoint(tmp_path / "m.mfam", b.download_params())
    V.save_state(tmp_path / "s.mfak", b.download_state())
    b.close()
    Xr = V.load_dataset(tmp_path / "x.mfad")
    r = V.Session(C, Xr.shape[1], H, Cp, G, Xr)
    r.set_floor(floor)
    r.upload_params(V.load_checkpoint(tmp_path / "m.mfam"))
    r.upload_state(V.load_state(tmp_path / "s.mfak"))
    rest = [r.iterate(0, it)["F"] for it in range(4, 7)]
    r.close()
    assert first + rest == full


def test_async_upload_matches_sync(oracle, gpu):
    # vmfa_upload_data_async: the copy runs on a second stream, ordered after
    # the work already enqueued and before the first X consumer; with lookahead
    # off (vmfa_set_lookahead) the iteration is unchanged
    O, V = oracle, gpu
    X, _ = gaussian_problem(5000, 64, 20, 3, seed=8)
    X2 = (X + np.float32(0.25)).astype(np.float32)
    C, H, Cp, G = 30, 4, 3, 5
    out = []
    for asynchronous in (False, True):
        p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
        sess.variational_e_step(0, 0)
        sess.iterate(0, 1)
        sess.set_lookahead(not asynchronous)
        pinned = np.empty_like(X2)
        pinned[...] = X2
        sess.upload_data(pinned, asynchronous=asynchronous)  # replaces the rows the last iteration used
        r = sess.iterate(0, 2)
        r3 = sess.iterate(0, 3)
        out.append((r["F"], r3["F"], sess.download_state().K, sess.download_params().mu))
        sess.close()
    (a, a3, Ka, mua), (b, b3, Kb, mub) = out
    assert a == b and a3 == b3
    assert np.array_equal(Ka, Kb) and np.array_equal(mua, mub)


def test_staged_rows_match_sync_upload(oracle, gpu):
    # vmfa_stage_data_async / vmfa_swap_data (the pipelined row uploads of the
    # e2e loop): rows staged while an iteration runs and swapped in before the
    # next one give the same iterations as synchronous uploads, across several
    # swaps (both device buffers in turn, one cached graph per buffer)
    O, V = oracle, gpu
    X, _ = gaussian_problem(5000, 64, 20, 3, seed=8)
    Xs = [X, (X + np.float32(0.25)).astype(np.float32), (X - np.float32(0.5)).astype(np.float32)]
    C, H, Cp, G = 30, 4, 3, 5
    out = []
    for staged in (False, True):
        p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
        sess.variational_e_step(0, 0)
        sess.set_lookahead(False)
        pinned = [np.ascontiguousarray(x) for x in Xs]
        rs = []
        if staged:
            sess.stage_data(pinned[1])
        for it in range(1, 6):
            nxt = pinned[(it + 1) % 3]
            if staged:
                sess.swap_data()      # this iteration's rows: pinned[it % 3]
                sess.stage_data(nxt)  # the next iteration's, copied while this one runs
            else:
                sess.upload_data(pinned[it % 3])
            rs.append(sess.iterate(0, it)["F"])
        out.append((rs, sess.download_state().K, sess.download_params().mu))
        sess.close()
    (ra, Ka, mua), (rb, Kb, mub) = out
    assert ra == rb
    assert np.array_equal(Ka, Kb) and np.array_equal(mua, mub)


def test_upload_state_validates_K_on_device(gpu):
    # VarState::validate (estep.cpp:15-68): K rows sorted, distinct, in range
    V = gpu
    X, _ = gaussian_problem(500, 16, 6, 2, seed=3)
    p, st, floor, _ = V.initialize(X, 10, 2, 3, 4, seed=1)
    sess = V.Session(10, 16, 2, 3, 4, X)
    sess.set_floor(floor)
    sess.upload_params(p)
    sess.upload_state(st)  # valid
    bad = st.K.copy()
    bad[137] = bad[137][::-1]  # unsorted row
    with pytest.raises(V.VmfaError, match=r"InvalidArgument.*n=137"):
        sess.upload_state(V.State(bad, st.g, st.g_count))
    bad = st.K.copy()
    bad[42, 0] = 10  # out of range
    with pytest.raises(V.VmfaError, match=r"n=42"):
        sess.upload_state(V.State(bad, st.g, st.g_count))
    sess.close()


def test_config5_shape_h64(oracle, gpu):
    # BASELINE config 5's model shape (D = 768, H = 64, C' = 5, G = 20) at a
    # small N and C: caches, a teacher-forced E-step, the statistics (two column
    # passes + the separate E pass of k_stats) and update_params vs the oracle
    O, V = oracle, gpu
    X, _ = gaussian_problem(2000, 768, 8, 16, seed=21)
    C, H, Cp, G = 24, 64, 5, 20
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    k = O.precompute_all(p)
    got = sess.download_caches()
    for name in ("Lmat", "Sz", "logdet"):
        np.testing.assert_allclose(got[name], getattr(k, name), rtol=1e-9, atol=1e-12, err_msg=name)
    e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sess, X, p, st, 5, 0)
    compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
    _, _, _, resp = sess.download_estep()
    s_or = O.accumulate_suffstats(X, p, k, st_g.K, resp, threads=4)
    sess.accumulate_suffstats()
    s_g = sess.download_suffstats()
    np.testing.assert_allclose(s_g.E, s_or.E, rtol=1e-5, atol=1e-6 * np.abs(s_or.E).max())
    np.testing.assert_allclose(s_g.Y, s_or.Y, rtol=1e-5, atol=1e-6 * np.abs(s_or.Y).max())
    np.testing.assert_allclose(s_g.sq, s_or.sq, rtol=1e-5)
    sess.upload_suffstats(s_or)
    sess.update_params()
    p_g = sess.download_params()
    p_or = O.update_params(s_or, X.shape[0], p, floor)
    for f in ("pi", "mu", "lam", "psi"):
        np.testing.assert_allclose(getattr(p_g, f), getattr(p_or, f), rtol=1e-8, atol=1e-11, err_msg=f)
    k2 = O.precompute_all(p_or)
    got = sess.download_caches()
    for name in ("Lmat", "Sz", "logdet"):
        np.testing.assert_allclose(got[name], getattr(k2, name), rtol=1e-8, atol=1e-11, err_msg=name)
    F_g = sess.truncated_free_energy()
    F_or = O.truncated_free_energy(X, p_or, k2, st_g.K, threads=4)
    assert abs(F_g - F_or) <= 1e-5 * abs(F_or)
    sess.close()


@pytest.mark.parametrize("case", [dict(N=4000, D=64, C=100, H=4, Cp=3, G=5),
                                  dict(N=6000, D=256, C=300, H=8, Cp=5, G=10)])
def test_sparse_cooc_matches_dense(oracle, gpu, case, monkeypatch):
    """Block 3 on sparse (c, c~) lists (the large-C path, forced by
    VMFA_COOC=sparse) reproduces the dense rows' g bit for bit (exact integer
    sums), and the oracle's g outside near-ties."""
    O, V = oracle, gpu
    X, _ = gaussian_problem(case["N"], case["D"], max(case["C"] // 2, 2), min(case["H"], 4), seed=17)
    C, H, Cp, G = case["C"], case["H"], case["Cp"], case["G"]
    monkeypatch.delenv("VMFA_COOC", raising=False)
    p, st, floor, dense = _setup(O, V, X, C, H, Cp, G)
    monkeypatch.setenv("VMFA_COOC", "sparse")
    _, _, _, sparse = _setup(O, V, X, C, H, Cp, G)
    monkeypatch.delenv("VMFA_COOC", raising=False)
    assert sparse.cooc_sparse() and not dense.cooc_sparse()
    for it in range(3):
        Fd, Jd = dense.variational_e_step(5, it)
        Fs, Js = sparse.variational_e_step(5, it)
        a, b = dense.download_state(), sparse.download_state()
        assert Jd == Js and Fd == Fs
        assert np.array_equal(a.K, b.K) and np.array_equal(a.labels, b.labels)
        assert np.array_equal(a.g, b.g) and np.array_equal(a.g_count, b.g_count)
    # against the oracle (teacher-forced step)
    e_or, st_or, F, J, ret, st_g, k = _estep_both(O, V, sparse, X, p, st, 7, 5)
    compare_estep(O, e_or, st_or, F, J, ret, st_g, Cp)
    same_part = ~np.zeros(C, bool)
    for n in np.nonzero(np.any(st_g.K != st_or.K, axis=1) | (st_g.labels != st_or.labels))[0]:
        same_part[st_or.labels[n]] = same_part[st_g.labels[n]] = False
    assert not compare_g(st_g.g, st_g.g_count, st_or.g, st_or.g_count, e_or.dist, same_part)
    dense.close()
    sparse.close()


def test_sparse_cooc_multishard(gpu, oracle, monkeypatch):
    """Three row shards in sparse mode, the owner-routed list exchange done on
    the host (the all-to-all of paper_2501_12299_b200.exchange.route_lists,
    emulated in-process), must give the single dense context's K, g and joint
    counts bit for bit, iteration after iteration."""
    import torch
    from paper_2501_12299_b200.exchange import XCHG_G, XCHG_SCALARS, XCHG_STATS, device_view
    O, V = oracle, gpu
    X, _ = gaussian_problem(6000, 32, 20, 3, seed=23)
    C, H, Cp, G, W = 45, 3, 3, 5, 3
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
    monkeypatch.delenv("VMFA_COOC", raising=False)
    single = V.Session(C, 32, H, Cp, G, X)
    single.set_floor(floor)
    single.upload_params(to_vmfa_params(V, p))
    single.upload_state(to_vmfa_state(V, st))
    monkeypatch.setenv("VMFA_COOC", "sparse")
    N = X.shape[0]
    shards = []
    for r in range(W):
        a, b = r * N // W, (r + 1) * N // W
        s = V.Session(C, 32, H, Cp, G, X[a:b], n_offset=a, n_total=N)
        s.set_floor(floor)
        s.upload_params(to_vmfa_params(V, p))
        s.upload_state(V.State(st.K[a:b].copy(), st.g.copy(), st.g_count.copy()))
        shards.append(s)
    monkeypatch.delenv("VMFA_COOC", raising=False)

    def view(s, which):
        ptr, n, dt = s.exchange_buffer(which)
        return device_view(ptr, n, {0: "<i8", 1: "<f8", 2: "<i4"}[dt])

    def allreduce(which):
        vs = [view(s, which) for s in shards]
        tot = sum(vs[1:], vs[0].clone())
        for v in vs:
            v.copy_(tot)
        torch.cuda.synchronize()

    def cooc_exchange():
        sent = []
        for s in shards:
            (pk, pc, ph, pl), counts = s.cooc_local_list(W)
            n = int(counts.sum())
            arrs = [device_view(pk, n, "<i4").clone(), device_view(pc, n, "<i8").clone(),
                    device_view(ph, n, "<i8").clone(), device_view(pl, n, "<i8").clone()]
            sent.append((arrs, np.concatenate([[0], np.cumsum(counts)])))
        for r, s in enumerate(shards):  # rank r receives the r-th slice of every source, in source order
            got = [torch.cat([arrs[i][off[r]:off[r + 1]] for arrs, off in sent]) for i in range(4)]
            n = got[0].numel()
            torch.cuda.synchronize()
            s.cooc_select([int(t.data_ptr()) if n else 0 for t in got], n, r, W)
        allreduce(XCHG_G)

    for it in range(3):
        rep = single.iterate(3, it)
        for s in shards:
            s.phase_estep_local(3, it)
        cooc_exchange()
        for s in shards:
            s.phase_estep_finish()
            s.phase_stats_local()
        allreduce(XCHG_STATS)
        for s in shards:
            s.phase_update()
            s.phase_free_energy_local()
        allreduce(XCHG_SCALARS)
        Fe, J, F = shards[0].phase_scalars()
        assert J == rep["joints"]
        assert abs(F - rep["F"]) <= 1e-7 * abs(rep["F"])
        st1 = single.download_state()
        parts = [s.download_state() for s in shards]
        assert np.array_equal(np.concatenate([q.K for q in parts]), st1.K)
        for q in parts:
            assert np.array_equal(q.g, st1.g) and np.array_equal(q.g_count, st1.g_count)
    for s in shards + [single]:
        s.close()


@pytest.mark.parametrize("chunk", [0, 700])
def test_em_full_step_matches_oracle(oracle, gpu, chunk, monkeypatch):
    """em_full_step (mstep.cpp:164-208) on the device: log-likelihood and the
    full-posterior statistics vs the oracle (q from fp32-accurate log-joints:
    relative errors ~|dl|), then update_params from them; chunk > 0 splits the
    rows into several dense chunks whose statistics are summed."""
    O, V = oracle, gpu
    if chunk:
        monkeypatch.setenv("VMFA_EM_CHUNK", str(chunk))
    else:
        monkeypatch.delenv("VMFA_EM_CHUNK", raising=False)
    X, _ = gaussian_problem(3000, 64, 12, 4, seed=31)
    C, H, Cp, G = 24, 4, 3, 5
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    k = O.precompute_all(p)
    s_or, ll_or, j_or = O.em_full_step(X, p, k, threads=4)
    ll, j = sess.em_full_step()
    assert j == j_or == X.shape[0] * C
    assert abs(ll - ll_or) <= 1e-5 * abs(ll_or)
    s_g = sess.download_suffstats()
    np.testing.assert_allclose(s_g.Nc, s_or.Nc, rtol=2e-3, atol=1e-6 * X.shape[0])
    for f in ("E", "Y", "sq"):
        a, b = getattr(s_g, f), getattr(s_or, f)
        np.testing.assert_allclose(a, b, rtol=2e-3, atol=2e-4 * np.abs(b).max(), err_msg=f)
    sess.upload_suffstats(s_or)
    sess.update_params()
    p_or = O.update_params(s_or, X.shape[0], p, floor)
    np.testing.assert_allclose(sess.download_params().mu, p_or.mu, rtol=1e-9, atol=1e-12)
    sess.close()


def test_train_emmfa_loop_matches_oracle(oracle, gpu):
    """run_emmfa_loop's iterations (em_full_step, update_params, exact F) on the
    device vs the oracle, free-running from the same initialisation: F per
    iteration within 1e-4 relative."""
    O, V = oracle, gpu
    X, _ = gaussian_problem(2000, 32, 6, 3, seed=41)
    C, H = 8, 3
    p, st, floor, sess = _setup(O, V, X, C, H, 3, 4)
    cfg = V.TrainConfig(max_iters=6, epsilon=0.0, halt_on_max_iters=False)
    rep = V.train_emmfa(sess, cfg)
    k = O.precompute_all(p)
    for r in rep["iterations"]:
        s_or, _, _ = O.em_full_step(X, p, k, threads=4)
        p = O.update_params(s_or, X.shape[0], p, floor)
        k = O.precompute_all(p)
        f_or = O.exact_log_likelihood(X, p, k, threads=4)
        assert abs(r["F"] - f_or) <= 1e-4 * abs(f_or), (r["t"], r["F"], f_or)
    assert rep["joint_evals"] == len(rep["iterations"]) * X.shape[0] * C
    # halt_on_max_iters (the default): MaxIterExceeded, as run_emmfa_loop's
    # use_eq14 path (trainer.cpp:262-266)
    with pytest.raises(V.VmfaError, match="MaxIterExceeded"):
        V.train_emmfa(sess, V.TrainConfig(max_iters=2, epsilon=0.0))
    sess.close()


@pytest.mark.parametrize("C,m", [(12, 10), (40, 3), (5, 1)])
def test_afkmc2_seed_matches_oracle(oracle, gpu, C, m):
    """AFK-MC^2 seeding (seeding.cpp:60-121, the reference's default init) on
    the device: the same seed rows, the same stream state after the draws and
    the same squared-distance count as the oracle (bit-identical fp64
    distances by explicit fma in ascending d)."""
    O, V = oracle, gpu
    X, _ = gaussian_problem(2500, 24, 8, 2, seed=51)
    seed = O.hash_combine(3, O.INIT_SALT)
    s_or, st_or, n_or = O.afkmc2_seed(X, C, m, seed)
    sess = V.Session(C, X.shape[1], 2, 2, 2, X)
    s_g, st_g, n_g = sess.afkmc2_seed(C, m, seed)
    assert np.array_equal(s_g, s_or)
    assert np.array_equal(st_g, st_or)
    assert n_g == n_or
    sess.close()


def test_afkmc2_degenerate_data(gpu, oracle):
    """Fewer distinct rows than seeds: DegenerateData on both sides (seeding.cpp:65-67)."""
    O, V = oracle, gpu
    X = np.repeat(np.arange(4, dtype=np.float32)[:, None], 8, axis=1)
    X = np.repeat(X, 50, axis=0)
    with pytest.raises(O.OracleError):
        O.afkmc2_seed(X, 6, 5, 1)
    sess = V.Session(6, 8, 1, 2, 2, X)
    with pytest.raises(V.VmfaError):
        sess.afkmc2_seed(6, 5, 1)
    sess.close()


def test_afkmc2_fallback_path(oracle, gpu):
    """Many duplicated rows: chains whose every proposal duplicates a chosen
    center take the farthest-point fallback (seeding.cpp:105-117); seeds,
    stream state and distance count still match the oracle bit for bit."""
    O, V = oracle, gpu
    rng = np.random.default_rng(4)
    base = rng.normal(0, 3, (7, 16)).astype(np.float32)
    X = np.repeat(base, 60, axis=0)
    rng.shuffle(X)
    seed = O.hash_combine(9, O.INIT_SALT)
    s_or, st_or, n_or = O.afkmc2_seed(X, 7, 2, seed)
    assert n_or > X.shape[0] + 2 * sum(range(1, 7))  # the fallback ran
    sess = V.Session(7, 16, 1, 2, 2, X)
    s_g, st_g, n_g = sess.afkmc2_seed(7, 2, seed)
    assert np.array_equal(s_g, s_or) and np.array_equal(st_g, st_or) and n_g == n_or
    sess.close()
