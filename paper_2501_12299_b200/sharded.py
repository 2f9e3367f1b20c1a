"""Sharded initialisation: the reference's ``initialize`` + ``init_varstate``
(trainer.cpp:32-47, 107-109) for a dataset whose rows are split over ranks,
without any rank holding all N rows.

The result is the one vmfa.initialize computes on the whole dataset: identical
seeds, parameters and K/g (bit for bit), and a floor equal up to the order of
the per-shard fp64 sums. The host pieces are in csrc/host/vmfa_host.cpp (see
include/vmfa_b200.h, "Sharded initialisation"); the collectives are the
caller's, through a ``Comm`` (torch.distributed, or a single process).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .abi import VmfaError, check, lib, ptr
from .vmfa import Params, State


class Comm:
    """Host-array collectives over torch.distributed (gloo on the host, or
    NCCL through device tensors); world 1 without a process group."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.device = device
        if self.dist and device is None:
            self.device = "cuda" if self.dist.get_backend(group) == "nccl" else "cpu"

    def allreduce(self, a: np.ndarray) -> np.ndarray:
        """Elementwise sum across ranks (a's dtype; int32 sums are exact)."""
        if self.world == 1:
            return a
        import torch
        t = torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def allgather(self, a: np.ndarray) -> list[np.ndarray]:
        """Every rank's array (lengths along axis 0 may differ)."""
        if self.world == 1:
            return [a]
        import torch
        n = torch.tensor([a.shape[0]], dtype=torch.int64, device=self.device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        ns = [int(v.item()) for v in ns]
        m = max(ns)
        pad = np.zeros((m,) + a.shape[1:], a.dtype)
        pad[:a.shape[0]] = a
        t = torch.from_numpy(pad).to(self.device)
        out = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy()[:k] for o, k in zip(out, ns)]


def _moments(X, mean=None, threads=0):
    out = np.zeros(X.shape[1])
    check(lib().vmfa_host_moments(ptr(X), X.shape[0], X.shape[1],
                                  None if mean is None else ptr(np.ascontiguousarray(mean, np.float64)),
                                  ptr(out), threads))
    return out


def variance_and_floor(X_local: np.ndarray, N: int, comm: Comm, threads: int = 0):
    """per_dimension_variance (dataset.cpp:22-35) as two moment all-reduces
    (the reference's two passes, with the global mean), and variance_floor
    (dataset.cpp:37-39)."""
    mean = comm.allreduce(_moments(X_local, None, threads)) / N
    var = comm.allreduce(_moments(X_local, mean, threads)) / N
    return var, np.maximum(1e-6 * var, 1e-8)


def distinct_rows_at_least(X_local: np.ndarray, C_: int, comm: Comm) -> bool:
    """count_distinct_rows(data, C) >= C (seeding.cpp:16-32, 127-129): the
    union of every shard's first C distinct rows, by 128-bit digests."""
    out = np.zeros((C_, 2), np.uint64)
    n = C.c_int64()
    check(lib().vmfa_host_distinct_hashes(ptr(X_local), X_local.shape[0], X_local.shape[1], C_, ptr(out),
                                          C.byref(n)))
    allh = np.concatenate(comm.allgather(out[:n.value].view(np.int64)))
    return len(np.unique(allh.view([("a", np.int64), ("b", np.int64)]))) >= C_


def seed_draws(seed: int, N: int, first: int, count: int) -> np.ndarray:
    out = np.zeros(count, np.int64)
    check(lib().vmfa_seed_draws(seed, N, first, count, ptr(out)))
    return out


def random_points_seed(X_local: np.ndarray, n0: int, N: int, C_: int, seed: int, comm: Comm):
    """random_points_seed (seeding.cpp:123-149) over sharded rows: the draws
    are replayed in order; the rows they name are fetched from their owners
    (an integer-sum all-reduce of the bit patterns: exact) and rejected as in
    the reference (already used, or equal to a chosen row under float ==).
    Returns (seed rows, their contents C x D, draws consumed)."""
    D = X_local.shape[1]
    n1 = n0 + X_local.shape[0]
    if not distinct_rows_at_least(X_local, C_, comm):
        raise VmfaError(8, "fewer distinct rows than requested seeds")
    used = set()
    chosen = {}
    seeds, rows_out = [], []
    first = 0
    consumed = None
    while consumed is None:
        batch = max(64, 2 * (C_ - len(seeds)))
        draws = seed_draws(seed, N, first, batch)
        need = np.unique(draws)
        rows = np.zeros((len(need), D), np.float32)
        mine = (need >= n0) & (need < n1)
        rows[mine] = X_local[need[mine] - n0]
        rows = comm.allreduce(rows.view(np.int32)).view(np.float32)
        where = {int(i): k for k, i in enumerate(need)}
        for k, i in enumerate(draws):
            i = int(i)
            if i in used:
                continue
            r = rows[where[i]]
            key = (r + np.float32(0.0)).tobytes()  # -0.0 == +0.0, as the reference's compare
            used.add(i)
            if key not in chosen:
                chosen[key] = i
                seeds.append(i)
                rows_out.append(r)
                if len(seeds) == C_:
                    consumed = first + k + 1
                    break
        first += batch
    return np.asarray(seeds, np.int64), np.ascontiguousarray(np.stack(rows_out)), consumed


def initialize_sharded(X_local: np.ndarray, n0: int, N: int, C_: int, H: int, Cprime: int, G: int,
                       seed: int = 0, scale: float = 0.1, loading_init: int = 1, comm: Comm | None = None,
                       threads: int = 0):
    """vmfa.initialize for the rows [n0, n0 + len(X_local)) of an N-row dataset
    held by this rank. Returns (params, state with the local K rows, floor,
    seeds) -- the same values on every rank, K aside."""
    comm = comm or Comm()
    X_local = np.ascontiguousarray(X_local, np.float32)
    D = X_local.shape[1]
    if not (1 <= C_ <= N and 1 <= H <= D and 1 <= Cprime <= C_ and 1 <= G <= C_):
        raise VmfaError(1, "initialize_sharded: invalid sizes")
    var, floor = variance_and_floor(X_local, N, comm, threads)
    seeds, srows, consumed = random_points_seed(X_local, n0, N, C_, seed, comm)
    rows = X_local.shape[0]
    p = Params(np.zeros(C_), np.zeros((C_, D)), np.zeros((C_, H, D)), np.zeros((C_, D)))
    st = State(np.zeros((rows, Cprime), np.int32), np.zeros((C_, G), np.int32), np.zeros(C_, np.int32),
               np.zeros(rows, np.int32))
    check(lib().vmfa_host_init_shard(N, D, C_, H, Cprime, G, seed, scale, loading_init, ptr(var), ptr(floor),
                                     ptr(seeds), ptr(srows), consumed, n0, rows, ptr(p.pi), ptr(p.mu),
                                     ptr(p.lam), ptr(p.psi), ptr(st.K), ptr(st.g), ptr(st.g_count)))
    return p, st, floor, seeds


__all__ = ["Comm", "initialize_sharded", "variance_and_floor", "random_points_seed", "seed_draws"]
