"""Multi-rank host logic on CPU (torch.distributed, gloo, world_size 2).

The B200 path shards rows over ranks and exchanges (i) the block-3
co-occurrence table and (ii) the sufficient statistics with all-reduces
(include/vmfa_b200.h phase API). This test runs the same
algebra with the fp64 oracle per shard: each rank runs the E-step on rows
[r*N/p, (r+1)*N/p) with the GLOBAL row index keying the extra candidate
(rng.hpp:91-98), all-reduces the dense (count, sum) co-occurrence table and the
statistics, and must reproduce the unsharded step: identical joint counts, K
rows, labels and g; F and the statistics equal to rounding; and the updated
parameters equal to rounding. The fixed-point encoding used on the GPU makes
the co-occurrence sums exact integers, checked here for order independence.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import gaussian_problem

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def select_g(cnt, ssum, G):
    """update_g (estep.cpp:204-220) from a dense per-component table."""
    C = cnt.shape[0]
    g = np.full((C, G), -1, np.int32)
    gc = np.zeros(C, np.int32)
    for c in range(C):
        keys = np.nonzero(cnt[c] > 0)[0]
        avg = ssum[c, keys] / cnt[c, keys]
        order = np.lexsort((keys, avg))[: G - 1]
        row = np.sort(np.concatenate([[c], keys[order]]))
        g[c, :len(row)] = row
        gc[c] = len(row)
    return g, gc


def _worker(rank, port, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    X, _ = gaussian_problem(1200, 8, 10, 2, seed=4)
    C, H, Cp, G = 16, 2, 3, 4
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=1, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    N = X.shape[0]
    a, b = rank * N // WORLD, (rank + 1) * N // WORLD
    shard = O.State(st.K[a:b].copy(), st.g.copy(), st.g_count.copy())
    e = O.variational_e_step(X[a:b], p, k, shard, 9, 3, threads=1, dump_distances=True, n_offset=a)
    # co-occurrence exchange: dense table, all-reduced
    cnt = np.zeros((C, C))
    ssum = np.zeros((C, C))
    dc, dct, ds, dn = e.dist
    cnt[dc, dct] = dn
    ssum[dc, dct] = ds
    t_cnt, t_sum = torch.from_numpy(cnt), torch.from_numpy(ssum)
    dist.all_reduce(t_cnt)
    dist.all_reduce(t_sum)
    g, gc = select_g(t_cnt.numpy(), t_sum.numpy(), G)
    # scalars
    sc = torch.tensor([e.F, float(e.joints)], dtype=torch.float64)
    dist.all_reduce(sc)
    # statistics with the pre-update caches and the shard's new K / resp
    s = O.accumulate_suffstats(X[a:b], p, k, shard.K, e.resp)
    flat = torch.from_numpy(np.concatenate([s.Nc, s.Y.ravel(), s.E.ravel(), s.sq.ravel()]))
    dist.all_reduce(flat)
    Ks = [torch.zeros((N // WORLD + 1, Cp), dtype=torch.int32) for _ in range(WORLD)]
    kpad = torch.zeros((N // WORLD + 1, Cp), dtype=torch.int32)
    kpad[: b - a] = torch.from_numpy(shard.K)
    dist.all_gather(Ks, kpad)
    if rank == 0:
        ret["g"], ret["gc"] = g, gc
        ret["F"], ret["J"] = float(sc[0]), int(sc[1])
        ret["stats"] = flat.numpy()
        ret["K"] = np.concatenate([Ks[r][: (r + 1) * N // WORLD - r * N // WORLD].numpy() for r in range(WORLD)])
    dist.destroy_process_group()


def test_two_rank_shard_algebra_matches_single(oracle):
    O = oracle
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(_free_port(), ret), nprocs=WORLD, join=True)
    X, _ = gaussian_problem(1200, 8, 10, 2, seed=4)
    C, H, Cp, G = 16, 2, 3, 4
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=1, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    e = O.variational_e_step(X, p, k, st, 9, 3, threads=1, dump_distances=True)
    assert ret["J"] == e.joints
    assert abs(ret["F"] - e.F) <= 1e-12 * abs(e.F)
    assert np.array_equal(ret["K"], st.K)
    assert np.array_equal(ret["gc"], st.g_count)
    assert np.array_equal(ret["g"], st.g)
    s = O.accumulate_suffstats(X, p, k, st.K, e.resp)
    single = np.concatenate([s.Nc, s.Y.ravel(), s.E.ravel(), s.sq.ravel()])
    np.testing.assert_allclose(ret["stats"], single, rtol=1e-12, atol=1e-12)


def to_fixed(v):
    """Host restatement of the device's fixed-point split (vmfa_kernels.cu
    to_fixed): value = hi * 2^-10 + lo * 2^-30, hi/lo int64, |value| <= 2^40."""
    v = float(np.clip(v, -2.0 ** 40, 2.0 ** 40))
    y = v * 1024.0
    f = np.floor(y)
    return int(f), int((y - f) * 2.0 ** 20)


def test_fixed_point_sums_are_order_and_partition_independent():
    rng = np.random.default_rng(0)
    vals = rng.normal(0, 50, 5000) * rng.choice([1e-3, 1, 1e3], 5000)
    parts = [to_fixed(v) for v in vals]
    hi = sum(p[0] for p in parts)
    lo = sum(p[1] for p in parts)
    perm = rng.permutation(len(parts))
    shard = [parts[i] for i in perm]
    hi2 = sum(p[0] for p in shard[:1234]) + sum(p[0] for p in shard[1234:])
    lo2 = sum(p[1] for p in shard[:1234]) + sum(p[1] for p in shard[1234:])
    assert (hi, lo) == (hi2, lo2)
    exact = hi / 1024.0 + lo / 2.0 ** 30
    assert abs(exact - vals.sum()) <= 1e-9 * np.abs(vals).sum()
    # the range: terms up to 2^40 in magnitude (a floored psi makes v^2/psi
    # huge), ~1e6 of them, still exact and order independent
    big = rng.uniform(-2.0 ** 40, 2.0 ** 40, 4096) * rng.choice([1e-9, 1.0], 4096)
    parts = [to_fixed(v) for v in big]
    hi, lo = sum(p[0] for p in parts), sum(p[1] for p in parts)
    assert abs(hi) < 2 ** 63 and 0 <= lo < 2 ** 63
    assert abs((hi / 1024.0 + lo / 2.0 ** 30) - float(np.sum(big))) <= 1e-12 * np.abs(big).sum()


def _sparse_worker(rank, port, ret):
    """The sparse co-occurrence exchange protocol of
    paper_2501_12299_b200.exchange (owner-routed lists via route_lists, owner
    reduce + select, int32 all-reduce of the selected rows) on the oracle's
    per-shard block-3 accumulators."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    from paper_2501_12299_b200.exchange import owner_ranges, route_lists
    X, _ = gaussian_problem(1500, 8, 12, 2, seed=6)
    C, H, Cp, G = 21, 2, 3, 4
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=2, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    N = X.shape[0]
    a, b = rank * N // WORLD, (rank + 1) * N // WORLD
    shard = O.State(st.K[a:b].copy(), st.g.copy(), st.g_count.copy())
    e = O.variational_e_step(X[a:b], p, k, shard, 4, 2, threads=1, dump_distances=True, n_offset=a)
    dc, dct, ds, dn = e.dist
    kb = int(C).bit_length()
    key = (dc.astype(np.int64) << kb) | dct.astype(np.int64)
    order = np.argsort(key, kind="stable")
    key, cnt, ssum, cc = key[order], dn[order].astype(np.int64), ds[order], dc[order]
    own = owner_ranges(C, WORLD)
    counts = [int(((cc >= lo) & (cc < hi)).sum()) for lo, hi in own]
    (rk, rn, rs), rc = route_lists([torch.from_numpy(key.astype(np.int32)), torch.from_numpy(cnt),
                                    torch.from_numpy(ssum)], counts)
    rk, rn, rs = rk.numpy().astype(np.int64), rn.numpy(), rs.numpy()
    # owner: reduce by key, select g for its components (rows of others stay 0)
    cnt_t, sum_t = np.zeros((C, C)), np.zeros((C, C))
    np.add.at(cnt_t, (rk >> kb, rk & ((1 << kb) - 1)), rn)
    np.add.at(sum_t, (rk >> kb, rk & ((1 << kb) - 1)), rs)
    g_all, gc_all = select_g(cnt_t, sum_t, G)
    lo, hi = own[rank]
    g = np.zeros((C, G), np.int32)
    gc = np.zeros(C, np.int32)
    g[lo:hi], gc[lo:hi] = g_all[lo:hi], gc_all[lo:hi]
    assert (rk >> kb).min(initial=lo) >= lo and (rk >> kb).max(initial=lo) < max(hi, lo + 1)
    buf = torch.from_numpy(np.concatenate([g.ravel(), gc]))
    dist.all_reduce(buf)
    out = buf.numpy()
    if rank == 0:
        ret["g"], ret["gc"] = out[:C * G].reshape(C, G), out[C * G:]
        ret["sent"], ret["recv"] = counts, rc
    dist.destroy_process_group()


def test_sparse_cooc_exchange_protocol(oracle):
    """Owner-routed sparse lists reproduce the unsharded E-step's g."""
    O = oracle
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_sparse_worker, args=(_free_port(), ret), nprocs=WORLD, join=True)
    X, _ = gaussian_problem(1500, 8, 12, 2, seed=6)
    C, H, Cp, G = 21, 2, 3, 4
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=2, scale=0.1, loading_init=1)
    k = O.precompute_all(p)
    O.variational_e_step(X, p, k, st, 4, 2, threads=1)
    assert sum(ret["recv"]) > 0 and sum(ret["sent"]) > 0
    assert np.array_equal(ret["gc"], st.g_count)
    assert np.array_equal(ret["g"], st.g)


def _init_worker(rank, port, ret, world, case):
    """initialize_sharded on rank-local rows only (gloo): each rank generates
    its own shard of the BASELINE generator's rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2501_12299_b200 import vmfa as V
    from paper_2501_12299_b200.sharded import Comm, initialize_sharded
    N = case["N"]
    a, b = rank * N // world, (rank + 1) * N // world
    X = V.gen_synthetic(V.synth_spec(case["cfg"], N=N), a, b)
    if case.get("dups"):  # duplicated rows exercise the duplicate rejection across shards
        X[::3] = V.gen_synthetic(V.synth_spec(case["cfg"], N=N), 0, 1)
    p, st, floor, seeds = initialize_sharded(X, a, N, case["C"], case["H"], case["Cp"], case["G"], seed=5,
                                             comm=Comm())
    ret[rank] = dict(pi=p.pi, mu=p.mu, lam=p.lam, psi=p.psi, K=st.K, g=st.g, gc=st.g_count, floor=floor,
                     seeds=seeds)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, dict(cfg=1, N=3000, C=100, H=4, Cp=3, G=5)),
    (3, dict(cfg=2, N=2500, C=300, H=8, Cp=5, G=10)),
    (2, dict(cfg=1, N=1500, C=60, H=2, Cp=3, G=4, dups=True)),
])
def test_sharded_initialize_matches_whole_dataset(vmfa, world, case):
    """Floor by moment all-reduces, seeds by draw replay + owner row fetch,
    init_varstate replayed per rank: identical to vmfa.initialize on all rows."""
    V = vmfa
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_init_worker, args=(_free_port(), ret, world, case), nprocs=world, join=True)
    N = case["N"]
    X = V.gen_synthetic(V.synth_spec(case["cfg"], N=N))
    if case.get("dups"):
        for r in range(world):
            a, b = r * N // world, (r + 1) * N // world
            X[a:b][::3] = X[0]
    p, st, floor, seeds = V.initialize(X, case["C"], case["H"], case["Cp"], case["G"], seed=5)
    for r in range(world):
        got = ret[r]
        assert np.array_equal(got["seeds"], seeds)
        for f in ("pi", "mu", "lam"):
            assert np.array_equal(got[f], getattr(p, f)), f
        np.testing.assert_allclose(got["psi"], p.psi, rtol=1e-12)
        np.testing.assert_allclose(got["floor"], floor, rtol=1e-12)
        assert np.array_equal(got["g"], st.g) and np.array_equal(got["gc"], st.g_count)
    K = np.concatenate([ret[r]["K"] for r in range(world)])
    assert np.array_equal(K, st.K)
