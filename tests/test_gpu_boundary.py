"""The reference API pieces beyond the fused iteration, on the device through
the C-ABI, against the oracle:
  * log_joint (model.hpp:83-86) in fp64;
  * the E-step's per-operation functions (estep.hpp:82-117) fed the oracle's
    own inputs: search spaces, update_k, hard_partition, accumulate_distances
    (fp64 sums in the reference's per-key order: bit-identical), update_g and
    responsibilities_row reproduce the oracle's E-step outputs exactly;
  * accumulate_suffstats with caller K / resp (mstep.hpp:27-31) and
    truncated_free_energy with caller ksets (model.hpp:116-119), driven by the
    fit_fa_per_cluster loop of kmeans.cpp:195-210 from C++ (tests/cpp/fit_fa.cpp).
"""
import os
import subprocess

import numpy as np
import pytest

from _helpers import gaussian_problem, to_vmfa_params, to_vmfa_state

pytestmark = pytest.mark.gpu


def _setup(O, V, X, C, H, Cp, G, seed=0):
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=seed, scale=0.1, loading_init=1)
    sess = V.Session(C, X.shape[1], H, Cp, G, X)
    sess.set_floor(floor)
    sess.upload_params(to_vmfa_params(V, p))
    sess.upload_state(to_vmfa_state(V, st))
    return p, st, floor, sess


def test_log_joint_matches_oracle(oracle, gpu):
    O, V = oracle, gpu
    X, _ = gaussian_problem(600, 40, 8, 3, seed=2)
    C, H = 12, 5
    p, st, floor, sess = _setup(O, V, X, C, H, 2, 3)
    p.pi[3] = 0.0
    p.pi /= p.pi.sum()
    sess.upload_params(to_vmfa_params(V, p))
    k = O.precompute_all(p)
    rng = np.random.default_rng(0)
    comp = rng.integers(0, C, 500).astype(np.int32)
    rows = rng.integers(0, X.shape[0], 500)
    got = sess.log_joint(X[rows], comp)
    want = np.array([O.log_joint(k, p.mu, int(c), X[r]) for r, c in zip(rows, comp)])
    fin = np.isfinite(want)
    assert np.all(np.isinf(got[~fin])) and (~fin).any()
    np.testing.assert_allclose(got[fin], want[fin], rtol=1e-12, atol=1e-9)
    sess.close()


@pytest.mark.parametrize("mode", [0, 1])
def test_per_operation_pieces_reproduce_the_estep(oracle, gpu, mode):
    O, V = oracle, gpu
    X, _ = gaussian_problem(3000, 24, 20, 3, seed=8)
    C, H, Cp, G = 40, 3, 3, 5
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    p.pi[[4, 17]] = 0.0  # frozen candidates are skipped by block 3
    p.pi /= p.pi.sum()
    sess.upload_params(to_vmfa_params(V, p))
    k = O.precompute_all(p)
    st_or = st.copy()
    e = O.variational_e_step(X, p, k, st_or, 9, 4, mode=mode, threads=4, dump_distances=True)
    # build_search_space: the oracle's retained indices are S(n) in insertion order
    cnt, idx = sess.build_search_space(9, 4)
    assert np.array_equal(cnt, e.count) and np.array_equal(idx, e.idx)
    extras = np.array([O.uniform_component(9, 4, n, C) for n in range(X.shape[0])], np.int32)
    cnt2, idx2 = sess.build_search_space(extras=extras)
    assert np.array_equal(idx2, e.idx)
    # update_k on the oracle's retained joints -> the oracle's new K
    Kn = sess.update_k(e.count, e.idx, e.lj)
    assert np.array_equal(Kn, st_or.K)
    # hard_partition -> labels; the partition lists ascending rows per label
    lab, off, ent = sess.hard_partition(Kn, e.count, e.idx, e.lj)
    assert np.array_equal(lab, st_or.labels)
    assert off[0] == 0 and off[-1] == X.shape[0]
    for c in range(C):
        rows = ent[off[c]:off[c + 1]]
        assert np.all(np.diff(rows) > 0) and np.all(lab[rows] == c)
    # accumulate_distances: bit-identical to the oracle's (same fp64 order)
    dc, dct, ds, dn = sess.accumulate_distances(mode, off, ent, e.count, e.idx, e.lj, p.pi)
    oc, oct_, os_, on = e.dist
    assert np.array_equal(dc, oc) and np.array_equal(dct, oct_) and np.array_equal(dn, on)
    assert np.array_equal(ds, os_), float(np.abs(ds - os_).max())
    # update_g -> the oracle's g
    g, gc = sess.update_g(dc, dct, ds, dn)
    assert np.array_equal(gc, st_or.g_count) and np.array_equal(g, st_or.g)
    # responsibilities_row over the new K's log-joints
    lk = np.array([[e.lj[n][e.idx[n] == c][0] for c in Kn[n]] for n in range(X.shape[0])])
    np.testing.assert_allclose(sess.responsibilities(lk), e.resp, rtol=1e-13, atol=1e-300)
    with pytest.raises(V.VmfaError, match="InsufficientCandidates"):
        short = e.count.copy()
        short[5] = Cp - 1
        sess.update_k(short, e.idx, e.lj)
    sess.close()


def test_suffstats_and_free_energy_with_caller_state(oracle, gpu):
    O, V = oracle, gpu
    X, _ = gaussian_problem(2500, 32, 10, 3, seed=12)
    C, H, Cp, G = 16, 3, 3, 4
    p, st, floor, sess = _setup(O, V, X, C, H, Cp, G)
    k = O.precompute_all(p)
    rng = np.random.default_rng(4)
    K = np.sort(np.stack([rng.choice(C, Cp, replace=False) for _ in range(X.shape[0])]), axis=1).astype(np.int32)
    resp = rng.dirichlet(np.ones(Cp), X.shape[0])
    s_g = sess.accumulate_suffstats_k(K, resp)
    s_o = O.accumulate_suffstats(X, p, k, K, resp, threads=4)
    for f in ("Nc", "E", "Y", "sq"):
        np.testing.assert_allclose(getattr(s_g, f), getattr(s_o, f), rtol=1e-5, atol=1e-6 * np.abs(getattr(s_o, f)).max())
    F_g = sess.truncated_free_energy_k(K)
    F_o = O.truncated_free_energy(X, p, k, K, threads=4)
    assert abs(F_g - F_o) <= 1e-6 * abs(F_o)
    bad = K.copy()
    bad[3] = bad[3][::-1]
    with pytest.raises(V.VmfaError, match="InvalidArgument"):
        sess.truncated_free_energy_k(bad)
    sess.close()


def test_fit_fa_per_cluster_loop_from_cpp(oracle, gpu, tmp_path):
    """kmeans.cpp:195-210 through include/vmfa_b200.hpp (C++): F per
    iteration and the fitted single-component FA match the oracle running the
    same calls; the truncated-F tally counts N C' joints per call."""
    from test_abi_host import build_fit_fa
    O, V = oracle, gpu
    X, _ = gaussian_problem(1500, 20, 1, 4, seed=31)
    N, D, H = X.shape[0], X.shape[1], 4
    floor = O.variance_floor(X)
    var = O.per_dimension_variance(X)
    rng = np.random.default_rng(5)
    fa = O.Params(np.ones(1), X.mean(axis=0, dtype=np.float64)[None, :], rng.uniform(0, 1, (1, H, D)),
                  np.maximum(var, floor)[None, :])
    V.save_dataset(tmp_path / "cell.mfad", X)
    V.save_checkpoint(tmp_path / "fa.mfam", to_vmfa_params(V, fa))
    floor.astype(np.float64).tofile(tmp_path / "floor.bin")
    exe = build_fit_fa(tmp_path)
    r = subprocess.run([str(exe), str(tmp_path / "cell.mfad"), str(tmp_path / "fa.mfam"), str(tmp_path / "floor.bin"),
                        "60", "1e-6", str(tmp_path / "out.mfam")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = [l.split() for l in r.stdout.strip().splitlines()]
    K = np.zeros((N, 1), np.int32)
    resp = np.ones((N, 1))
    k = O.precompute_all(fa)
    prev, rows = np.nan, []
    for it in range(60):  # the reference's loop, on the oracle
        s = O.accumulate_suffstats(X, fa, k, K, resp, threads=4)
        fa = O.update_params(s, N, fa, floor)
        k = O.precompute_all(fa)
        F = O.truncated_free_energy(X, fa, k, K, threads=4)
        rows.append(F)
        if np.isfinite(prev) and abs(F - prev) < 1e-6 * abs(prev):
            break
        prev = F
    assert len(got) == len(rows)
    for (it, Fg, joints), Fo in zip(got, rows):
        assert abs(float(Fg) - Fo) <= 1e-4 * abs(Fo), (it, Fg, Fo)
        assert int(joints) == (int(it) + 1) * N  # EvalCounter: N C' per truncated F
    out = V.load_checkpoint(tmp_path / "out.mfam")
    np.testing.assert_allclose(out.mu, fa.mu, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(out.psi, fa.psi, rtol=1e-4)
    np.testing.assert_allclose(out.lam, fa.lam, rtol=1e-3, atol=1e-4 * np.abs(fa.lam).max())


@pytest.mark.parametrize("cooc", ["dense", "sparse"])
def test_torchrun_two_ranks_match_one(gpu, tmp_path, cooc):
    """bench.py's multi-rank path (one process per rank, the phase API, the
    co-occurrence and statistics exchanges of paper_2501_12299_b200.exchange)
    under torchrun with 2 ranks on this one GPU (gloo collectives: host-staged,
    no kernel waits on another rank), against the same run on 1 rank: the
    sharded generation / floor / initialisation and every iteration give the
    single-rank K rows and g exactly, and F to rounding."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    if cooc == "sparse":
        env["VMFA_COOC"] = "sparse"
    common = ["bench.py", "--config", "2", "--rows", "12000", "--steps", "2", "--warmup", "1", "--no-e2e",
              "--no-cpu-baseline", "--no-exact-ll", "--backend", "gloo"]
    one = subprocess.run([sys.executable] + common + ["--dump-state", str(tmp_path / "one")], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert one.returncode == 0, one.stderr[-2000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 500))] + common +
                         ["--gpus", "2", "--dump-state", str(tmp_path / "two")], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert two.returncode == 0, two.stderr[-3000:]
    line1 = json.loads(one.stdout.strip().splitlines()[-1])
    line2 = json.loads(two.stdout.strip().splitlines()[-1])
    assert line2["n_gpus"] == 2
    a = np.load(str(tmp_path / "one.rank0.npz"))
    r0, r1 = np.load(str(tmp_path / "two.rank0.npz")), np.load(str(tmp_path / "two.rank1.npz"))
    # the ranks' g are replicated exactly (exact integer co-occurrence sums)
    assert np.array_equal(r0["g"], r1["g"]) and np.array_equal(r0["mu"], r1["mu"])
    # against one rank: the statistics are summed in another grouping (fp64
    # rounding), so after several M-steps fp32 score roundings can flip rows
    # whose top-C' boundary is a near-tie -- all others agree
    K2 = np.concatenate([r0["K"], r1["K"]])
    same = np.mean(np.all(K2 == a["K"], axis=1))
    assert same >= 0.995, same
    assert np.mean(np.all(r0["g"] == a["g"], axis=1)) >= 0.99
    np.testing.assert_allclose(r0["J"], a["J"], rtol=1e-3)
    np.testing.assert_allclose(r0["F"], a["F"], rtol=1e-4)  # the north-star F tolerance
    np.testing.assert_allclose(r0["mu"], a["mu"], rtol=1e-3, atol=1e-3 * np.abs(a["mu"]).max())


@pytest.mark.parametrize("C", [200, 4000, 40000])
def test_partition_sort_at_scale(gpu, C):
    """The K1 inversion's hand-written stable radix sort (vmfa_sort.cu; one,
    two 8-bit passes) through hard_partition at 2M rows: labels are the
    first strict maximum of each K row's log-joints, and the partition equals
    numpy's stable argsort of the labels (rows ascending per component, the
    reference's push order, estep.cpp:169-172)."""
    V = gpu
    N, D, Cp, G = 2_000_000, 8, 3, 2
    rng = np.random.default_rng(C)
    sess = V.Session(C, D, 1, Cp, G, np.zeros((N, D), np.float32))
    S = sess.stride
    K = np.sort(np.stack([rng.choice(C, Cp, replace=False) for _ in range(256)]), axis=1)
    K = K[rng.integers(0, 256, N)].astype(np.int32)  # 256 distinct sorted rows, repeated
    idx = np.full((N, S), -1, np.int32)
    idx[:, :Cp] = K
    lj = np.zeros((N, S))
    lj[:, :Cp] = rng.integers(0, 4, (N, Cp)).astype(np.float64)  # ties: the first member wins
    count = np.full(N, Cp, np.int32)
    lab, off, ent = sess.hard_partition(K, count, idx, lj)
    want = K[np.arange(N), np.argmax(lj[:, :Cp], axis=1)]
    assert np.array_equal(lab, want)
    assert np.array_equal(ent, np.argsort(want, kind="stable").astype(np.int32))
    assert np.array_equal(off, np.searchsorted(np.sort(want), np.arange(C + 1)).astype(np.int32))
    sess.close()
