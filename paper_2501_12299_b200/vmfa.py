"""Python mirror of the reference's v-MFA API over libvmfa_b200.so.

Names and semantics follow /root/reference/proj/include/vmfa/:
  MfaParams (model.hpp:19-32)   -> Params
  VarState  (estep.hpp:17-29)   -> State
  SuffStats (mstep.hpp:14-22)   -> Stats
  variational_e_step (estep.hpp:125-130), accumulate_suffstats
  (mstep.hpp:27-31), update_params (mstep.hpp:39-41), precompute_all
  (model.hpp:76-78), truncated_free_energy (model.hpp:116-119)
  -> methods of Session, which owns one GPU context (one shard of the rows).
train_fixed mirrors train_vmfa's loop (trainer.cpp:111-186) with fixed counts.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from .abi import IterReport, SynthSpec, VmfaError, check, lib, ptr

KL, EUCLID = 0, 1  # DistanceMode (estep.hpp:12)


@dataclass
class Params:
    """MfaParams: pi (C,), mu (C,D), lam (C,H,D) = per-component D x H
    column-major blocks, psi (C,D) = the reference's ``dnoise``."""
    pi: np.ndarray
    mu: np.ndarray
    lam: np.ndarray
    psi: np.ndarray

    @property
    def C(self):
        return self.mu.shape[0]

    @property
    def D(self):
        return self.mu.shape[1]

    @property
    def H(self):
        return self.lam.shape[1]

    def copy(self):
        return Params(self.pi.copy(), self.mu.copy(), self.lam.copy(), self.psi.copy())


@dataclass
class State:
    """VarState: K (N,C') sorted rows, g (C,G) sorted rows -1 padded, g_count (C,)."""
    K: np.ndarray
    g: np.ndarray
    g_count: np.ndarray
    labels: np.ndarray = field(default=None)

    def copy(self):
        return State(self.K.copy(), self.g.copy(), self.g_count.copy(),
                     None if self.labels is None else self.labels.copy())


@dataclass
class Stats:
    Nc: np.ndarray
    Y: np.ndarray   # (C,H+1,D)
    E: np.ndarray   # (C,H+1,H+1)
    sq: np.ndarray  # (C,D)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def device_available() -> bool:
    return bool(lib().vmfa_device_available())


class Session:
    """One device context: rows [n_offset, n_offset + len(X)) of an n_total-row
    dataset, replicated parameters/caches, and the shard's variational state."""

    def __init__(self, C_: int, D: int, H: int, Cprime: int, G: int, X: np.ndarray,
                 n_offset: int = 0, n_total: int | None = None, device: int = 0,
                 stream: int | None = None):
        X = _c(X, np.float32)
        assert X.ndim == 2 and X.shape[1] == D
        self.C, self.D, self.H, self.Cp, self.G = C_, D, H, Cprime, G
        self.N = X.shape[0]
        self.n_offset = n_offset
        self.n_total = self.N + n_offset if n_total is None else n_total
        self.stride = min(Cprime * G + 1, C_)
        h = C.c_void_p()
        check(lib().vmfa_ctx_create(C.byref(h), device, C_, D, H, Cprime, G, self.N, n_offset,
                                    self.n_total, stream))
        self._h = h
        check(lib().vmfa_upload_data(h, ptr(X), 0, self.N))

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().vmfa_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def device_bytes(self) -> int:
        b = C.c_size_t()
        check(lib().vmfa_ctx_device_bytes(self._h, C.byref(b)))
        return b.value

    def upload_data(self, X: np.ndarray, row_begin: int = 0, asynchronous: bool = False):
        """Rows [row_begin, row_begin + len(X)) of this shard. asynchronous:
        vmfa_upload_data_async -- the copy overlaps the work enqueued next (X
        must stay unchanged until the next synchronising call; the session
        keeps a reference to it)."""
        X = _c(X, np.float32)
        if asynchronous:
            check(lib().vmfa_upload_data_async(self._h, ptr(X), row_begin, X.shape[0]))
            self._pending_x = X
        else:
            check(lib().vmfa_upload_data(self._h, ptr(X), row_begin, X.shape[0]))

    def stage_data(self, X: np.ndarray, row_begin: int = 0):
        """vmfa_stage_data_async: rows into the second device buffer on the copy
        stream (the next batch, while the current one is processed); X must
        stay unchanged until the next synchronising call."""
        X = _c(X, np.float32)
        check(lib().vmfa_stage_data_async(self._h, ptr(X), row_begin, X.shape[0]))
        self._staged_x = X

    def swap_data(self):
        """vmfa_swap_data: the staged rows become current."""
        check(lib().vmfa_swap_data(self._h))

    def set_lookahead(self, enable: bool):
        """vmfa_set_lookahead: truncated F from the next E-step's anchor pass
        (default) or from its own one-component pass (same value)."""
        check(lib().vmfa_set_lookahead(self._h, 1 if enable else 0))

    # -- params / caches
    def set_floor(self, floor):
        check(lib().vmfa_set_floor(self._h, ptr(_c(floor, np.float64))))

    def upload_params(self, p: Params):
        check(lib().vmfa_upload_params(self._h, ptr(_c(p.pi, np.float64)), ptr(_c(p.mu, np.float64)),
                                       ptr(_c(p.lam, np.float64)), ptr(_c(p.psi, np.float64))))

    def download_params(self, out: Params | None = None) -> Params:
        """Parameters into new arrays, or into `out` (e.g. pinned buffers reused per step)."""
        p = out if out is not None else Params(np.zeros(self.C), np.zeros((self.C, self.D)),
                                               np.zeros((self.C, self.H, self.D)), np.zeros((self.C, self.D)))
        check(lib().vmfa_download_params(self._h, ptr(p.pi), ptr(p.mu), ptr(p.lam), ptr(p.psi)))
        return p

    def precompute(self):
        bad = C.c_int(-1)
        check(lib().vmfa_precompute(self._h, C.byref(bad)))

    def download_caches(self):
        C_, D, H = self.C, self.D, self.H
        out = dict(U=np.zeros((C_, H, D)), Lmat=np.zeros((C_, H, H)), V=np.zeros((C_, D, H)),
                   Sz=np.zeros((C_, H, H)), inv_psi=np.zeros((C_, D)), logdet=np.zeros(C_),
                   log_pi=np.zeros(C_))
        check(lib().vmfa_download_caches(self._h, ptr(out["U"]), ptr(out["Lmat"]), ptr(out["V"]),
                                         ptr(out["Sz"]), ptr(out["inv_psi"]), ptr(out["logdet"]),
                                         ptr(out["log_pi"])))
        return out

    # -- state
    def upload_state(self, st: State):
        check(lib().vmfa_upload_state(self._h, ptr(_c(st.K, np.int32)), ptr(_c(st.g, np.int32)),
                                      ptr(_c(st.g_count, np.int32))))

    def download_state(self, out: State | None = None) -> State:
        """State into new arrays, or into `out` (labels included)."""
        st = out if out is not None else State(np.zeros((self.N, self.Cp), np.int32),
                                               np.zeros((self.C, self.G), np.int32),
                                               np.zeros(self.C, np.int32), np.zeros(self.N, np.int32))
        check(lib().vmfa_download_state(self._h, ptr(st.K), ptr(st.g), ptr(st.g_count),
                                        ptr(st.labels)))
        return st

    # -- hot path
    def variational_e_step(self, seed: int, iteration: int, mode: int = KL):
        F = C.c_double()
        J = C.c_uint64()
        check(lib().vmfa_estep(self._h, seed, iteration, mode, C.byref(F), C.byref(J)))
        return F.value, J.value

    def download_estep(self):
        N, S, Cp = self.N, self.stride, self.Cp
        cnt = np.zeros(N, np.int32)
        idx = np.zeros((N, S), np.int32)
        lj = np.zeros((N, S), np.float64)
        resp = np.zeros((N, Cp), np.float64)
        check(lib().vmfa_download_estep(self._h, ptr(cnt), ptr(idx), ptr(lj), ptr(resp)))
        return cnt, idx, lj, resp

    def arm_distance_dump(self):
        n = C.c_int64()
        check(lib().vmfa_download_distances(self._h, 0, None, None, None, None, C.byref(n)))

    def download_distances(self):
        n = C.c_int64()
        check(lib().vmfa_download_distances(self._h, 0, None, None, None, None, C.byref(n)))
        m = n.value
        c = np.zeros(m, np.int32)
        ct = np.zeros(m, np.int32)
        s = np.zeros(m, np.float64)
        k = np.zeros(m, np.int64)
        if m:
            check(lib().vmfa_download_distances(self._h, m, ptr(c), ptr(ct), ptr(s), ptr(k),
                                                C.byref(n)))
            m = n.value  # rows of split components merged
        return c[:m], ct[:m], s[:m], k[:m]

    def accumulate_suffstats(self):
        check(lib().vmfa_accumulate_suffstats(self._h))

    def download_suffstats(self) -> Stats:
        C_, D, H1 = self.C, self.D, self.H + 1
        s = Stats(np.zeros(C_), np.zeros((C_, H1, D)), np.zeros((C_, H1, H1)), np.zeros((C_, D)))
        check(lib().vmfa_download_suffstats(self._h, ptr(s.Nc), ptr(s.Y), ptr(s.E), ptr(s.sq)))
        return s

    def upload_suffstats(self, s: Stats):
        check(lib().vmfa_upload_suffstats(self._h, ptr(_c(s.Nc, np.float64)), ptr(_c(s.Y, np.float64)),
                                          ptr(_c(s.E, np.float64)), ptr(_c(s.sq, np.float64))))

    def update_params(self):
        bad = C.c_int(-1)
        check(lib().vmfa_update_params(self._h, C.byref(bad)))

    def truncated_free_energy(self) -> float:
        F = C.c_double()
        check(lib().vmfa_truncated_free_energy(self._h, C.byref(F)))
        return F.value

    # -- the reference's entry points with caller-supplied state / per-op pieces
    def accumulate_suffstats_k(self, K: np.ndarray, resp: np.ndarray) -> Stats:
        """accumulate_suffstats(params, caches, data, ksets, resp) (mstep.hpp:27-31)
        with the caller's K rows and responsibilities (the context's K becomes K)."""
        check(lib().vmfa_accumulate_suffstats_k(self._h, ptr(_c(K, np.int32)), ptr(_c(resp, np.float64))))
        return self.download_suffstats()

    def truncated_free_energy_k(self, K: np.ndarray) -> float:
        """truncated_free_energy(params, caches, data, ksets) (model.hpp:116-119)."""
        F = C.c_double()
        check(lib().vmfa_truncated_free_energy_k(self._h, ptr(_c(K, np.int32)), C.byref(F)))
        return F.value

    def log_joint(self, X: np.ndarray, comp: np.ndarray) -> np.ndarray:
        """log_joint (model.hpp:83-86) for rows X[i] and components comp[i], fp64."""
        X = _c(X, np.float32).reshape(-1, self.D)
        comp = _c(comp, np.int32)
        out = np.zeros(X.shape[0])
        check(lib().vmfa_log_joint(self._h, ptr(X), X.shape[0], ptr(comp), ptr(out)))
        return out

    def build_search_space(self, seed: int = 0, iteration: int = 0, extras: np.ndarray | None = None):
        """build_search_space (estep.hpp:82-84) for every row: (count, idx)."""
        cnt = np.zeros(self.N, np.int32)
        idx = np.zeros((self.N, self.stride), np.int32)
        check(lib().vmfa_build_search_space(self._h, seed, iteration,
                                            None if extras is None else ptr(_c(extras, np.int32)), ptr(cnt),
                                            ptr(idx)))
        return cnt, idx

    def update_k(self, count, idx, lj) -> np.ndarray:
        """update_k (estep.hpp:88-90) for every row."""
        K = np.zeros((self.N, self.Cp), np.int32)
        check(lib().vmfa_update_k(self._h, ptr(_c(count, np.int32)), ptr(_c(idx, np.int32)), ptr(_c(lj, np.float64)),
                                  ptr(K)))
        return K

    def hard_partition(self, K, count, idx, lj):
        """hard_partition (estep.hpp:94-97): (labels, partition offsets, rows)."""
        lab = np.zeros(self.N, np.int32)
        off = np.zeros(self.C + 1, np.int32)
        ent = np.zeros(self.N, np.int32)
        check(lib().vmfa_hard_partition(self._h, ptr(_c(K, np.int32)), ptr(_c(count, np.int32)),
                                        ptr(_c(idx, np.int32)), ptr(_c(lj, np.float64)), ptr(lab), ptr(off),
                                        ptr(ent)))
        return lab, off, ent

    def accumulate_distances(self, mode, part_off, part_ent, count, idx, lj, pi):
        """accumulate_distances (estep.hpp:103-106): (c, ct, sum, count) rows."""
        args = [ptr(_c(part_off, np.int32)), ptr(_c(part_ent, np.int32)), ptr(_c(count, np.int32)),
                ptr(_c(idx, np.int32)), ptr(_c(lj, np.float64)), ptr(_c(pi, np.float64))]
        n = C.c_int64()
        check(lib().vmfa_accumulate_distances(self._h, mode, *args, 0, None, None, None, None, C.byref(n)))
        m = n.value
        c, ct, sm, cn = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m), np.zeros(m, np.int64)
        check(lib().vmfa_accumulate_distances(self._h, mode, *args, m, ptr(c), ptr(ct), ptr(sm), ptr(cn),
                                              C.byref(n)))
        return c, ct, sm, cn

    def update_g(self, c, ct, sm, cn):
        """update_g (estep.hpp:111-112) for every component: (g, g_count)."""
        g = np.zeros((self.C, self.G), np.int32)
        gc = np.zeros(self.C, np.int32)
        check(lib().vmfa_update_g(self._h, len(c), ptr(_c(c, np.int32)), ptr(_c(ct, np.int32)),
                                  ptr(_c(sm, np.float64)), ptr(_c(cn, np.int64)), ptr(g), ptr(gc)))
        return g, gc

    def responsibilities(self, lj: np.ndarray) -> np.ndarray:
        """responsibilities_row (estep.hpp:116-117) for every row of lj."""
        lj = _c(lj, np.float64)
        out = np.zeros_like(lj)
        check(lib().vmfa_responsibilities(self._h, lj.shape[0], lj.shape[1], ptr(lj), ptr(out)))
        return out

    def exact_log_likelihood(self) -> float:
        """exact_log_likelihood (model.cpp:139-148) over this session's rows:
        sum_n log sum_c p(x_n, c) over all C components (dense tcgen05 pass)."""
        ll = C.c_double()
        check(lib().vmfa_exact_log_likelihood(self._h, C.byref(ll)))
        return ll.value

    def em_full_step(self):
        """em_full_step (mstep.cpp:164-208): full-posterior statistics over
        every (n, c) pair left in the session (update_params follows, as in
        run_emmfa_loop, trainer.cpp:228-233). Returns (log-likelihood, joints)."""
        ll = C.c_double()
        j = C.c_uint64()
        check(lib().vmfa_em_full_step(self._h, C.byref(ll), C.byref(j)))
        return ll.value, j.value

    def afkmc2_seed(self, C_: int, chain_length: int, stream_seed: int):
        """afkmc2_seed (seeding.cpp:60-121) on the device over this session's
        rows (the whole dataset). Returns (seed rows, stream state after,
        squared-distance count); init_params continues the stream."""
        seeds = np.zeros(C_, np.int64)
        state = np.zeros(4, np.uint64)
        cnt = C.c_uint64()
        check(lib().vmfa_afkmc2_seed(self._h, C_, chain_length, stream_seed, ptr(seeds), ptr(state),
                                     C.byref(cnt)))
        return seeds, state, cnt.value

    def iterate(self, seed: int, iteration: int, mode: int = KL) -> dict:
        r = IterReport()
        check(lib().vmfa_iterate(self._h, seed, iteration, mode, C.byref(r)))
        return dict(F_estep=r.free_energy_estep, F=r.free_energy, joints=r.joints,
                    empty=r.empty_components)

    # -- multi-GPU phases
    def exchange_buffer(self, which: int):
        p = C.c_void_p()
        n = C.c_size_t()
        dt = C.c_int()
        check(lib().vmfa_exchange_buffer(self._h, which, C.byref(p), C.byref(n), C.byref(dt)))
        return p.value, n.value, dt.value

    def cooc_sparse(self) -> bool:
        """vmfa_cooc_sparse: True when block 3 runs on sparse (c, c~) lists
        (C too large for the dense table, or VMFA_COOC=sparse at creation)."""
        v = C.c_int()
        check(lib().vmfa_cooc_sparse(self._h, C.byref(v)))
        return bool(v.value)

    def cooc_local_list(self, world: int):
        """vmfa_cooc_local_list: device pointers (key u32, cnt, hi, lo int64) of
        this rank's reduced list, sorted by key, and the entry count per owner
        rank (block ownership of components)."""
        ps = [C.c_void_p() for _ in range(4)]
        counts = np.zeros(world, np.int64)
        check(lib().vmfa_cooc_local_list(self._h, world, *[C.byref(q) for q in ps], ptr(counts)))
        return tuple(q.value for q in ps), counts

    def cooc_select(self, ptrs, n: int, rank: int, world: int):
        """vmfa_cooc_select: reduce the received lists (device pointers) and
        select g for this rank's components into the VMFA_XCHG_G buffer."""
        check(lib().vmfa_cooc_select(self._h, *[C.c_void_p(q) for q in ptrs], int(n), rank, world))

    def phase_estep_local(self, seed, it, mode=KL):
        check(lib().vmfa_phase_estep_local(self._h, seed, it, mode))

    def phase_estep_finish(self):
        check(lib().vmfa_phase_estep_finish(self._h))

    def phase_stats_local(self):
        check(lib().vmfa_phase_stats_local(self._h))

    def phase_update(self):
        bad = C.c_int(-1)
        check(lib().vmfa_phase_update(self._h, C.byref(bad)))

    def phase_free_energy_local(self):
        check(lib().vmfa_phase_free_energy_local(self._h))

    def phase_scalars(self):
        Fe, F = C.c_double(), C.c_double()
        J = C.c_uint64()
        check(lib().vmfa_phase_scalars(self._h, C.byref(Fe), C.byref(J), C.byref(F)))
        return Fe.value, J.value, F.value

    # -- profiling
    def profile(self, enable: bool = True):
        check(lib().vmfa_profile_enable(self._h, 1 if enable else 0))

    def kernel_times(self) -> dict:
        m = 16
        ms = np.zeros(m)
        la = np.zeros(m, np.int64)
        un = np.zeros(m, np.int64)
        n = C.c_int()
        check(lib().vmfa_kernel_times(self._h, m, ptr(ms), ptr(la), ptr(un), C.byref(n)))
        return {lib().vmfa_kernel_name(i).decode(): dict(ms=float(ms[i]), launches=int(la[i]),
                                                         units=int(un[i])) for i in range(n.value)}

    def scoring_work(self) -> dict:
        """vmfa_scoring_work: row visits, image / record bytes of the scoring launches."""
        w = np.zeros(8, np.int64)
        check(lib().vmfa_scoring_work(self._h, ptr(w), 8))
        return dict(anchor_visits=int(w[0]), extra_visits=int(w[1]), image_bytes=int(w[2]),
                    single_image_bytes=int(w[3]), record_bytes=int(w[4]), scorer=int(w[5]),
                    fp64_rescored=int(w[6]), tensor_rescored=int(w[7]))

    def stream(self) -> int:
        return lib().vmfa_ctx_stream(self._h)

    def synchronize(self):
        check(lib().vmfa_synchronize(self._h))


# ---------------------------------------------------------------- host helpers
# BASELINE.json configs: truth generator + fitted model.
CONFIGS = {
    1: dict(truth=dict(kind=0, N=20_000, D=64, C_true=100, H_true=4, dirichlet=0, mu_std=4.0,
                       lam_std=0.5, psi_lo=0.1, psi_hi=1.0),
            model=dict(C=100, H=4, Cprime=3, G=5, iters=20)),
    2: dict(truth=dict(kind=0, N=200_000, D=256, C_true=1000, H_true=8, dirichlet=1, mu_std=3.0,
                       lam_std=1 / np.sqrt(8), psi_lo=0.05, psi_hi=0.5),
            model=dict(C=1000, H=8, Cprime=5, G=10, iters=25)),
    3: dict(truth=dict(kind=1, N=1_000_000, D=784, C_true=4000, H_true=16, dirichlet=0,
                       lam_std=0.05, noise_std=0.05, img_w=28, img_h=28, img_c=1, blur_sigma=2.0),
            model=dict(C=4000, H=16, Cprime=5, G=10, iters=20)),
    4: dict(truth=dict(kind=0, N=10_000_000, D=256, C_true=10_000, H_true=8, dirichlet=1,
                       mu_std=3.0, lam_std=1 / np.sqrt(8), psi_lo=0.05, psi_hi=0.5),
            model=dict(C=10_000, H=8, Cprime=5, G=15, iters=15)),
    5: dict(truth=dict(kind=1, N=50_000_000, D=768, C_true=50_000, H_true=16, dirichlet=0,
                       lam_std=0.05, noise_std=0.05, img_w=16, img_h=16, img_c=3, blur_sigma=2.0),
            model=dict(C=50_000, H=64, Cprime=5, G=20, iters=10)),
}


def synth_spec(cfg: int, N: int | None = None, data_seed: int = 0, **over) -> SynthSpec:
    t = dict(CONFIGS[cfg]["truth"])
    t.update(over)
    sp = SynthSpec()
    sp.kind = t["kind"]
    sp.n_total = N if N is not None else t["N"]
    sp.D = t["D"]
    sp.C_true = t["C_true"]
    sp.H_true = t["H_true"]
    sp.dirichlet = t.get("dirichlet", 0)
    sp.mu_std = t.get("mu_std", 0.0)
    sp.lam_std = t.get("lam_std", 0.0)
    sp.psi_lo = t.get("psi_lo", 0.0)
    sp.psi_hi = t.get("psi_hi", 0.0)
    sp.noise_std = t.get("noise_std", 0.0)
    sp.img_w = t.get("img_w", 0)
    sp.img_h = t.get("img_h", 0)
    sp.img_c = t.get("img_c", 0)
    sp.blur_sigma = t.get("blur_sigma", 0.0)
    sp.data_seed = data_seed
    return sp


def gen_synthetic(spec: SynthSpec, row_begin: int = 0, row_end: int | None = None,
                  threads: int = 0, with_labels: bool = False):
    """Synthetic rows [row_begin, row_end) of a BASELINE config (host only)."""
    row_end = spec.n_total if row_end is None else row_end
    X = np.empty((row_end - row_begin, spec.D), np.float32)
    lab = np.empty(row_end - row_begin, np.int32) if with_labels else None
    check(lib().vmfa_gen_synthetic(C.byref(spec), row_begin, row_end, ptr(X), ptr(lab),
                                   threads or (os.cpu_count() or 1)))
    return (X, lab) if with_labels else X


def initialize(X: np.ndarray, C_: int, H: int, Cprime: int, G: int, seed: int = 0,
               scale: float = 0.1, loading_init: int = 1):
    """trainer.cpp:32-47 + :107-109 with random-points seeding (host only).
    Defaults follow BASELINE config 1's init: Lambda ~ N(0, 0.01) (scale 0.1,
    loading_init=1); loading_init=0, scale=1 is the reference's U[0,1)."""
    X = _c(X, np.float32)
    N, D = X.shape
    floor = np.zeros(D)
    p = Params(np.zeros(C_), np.zeros((C_, D)), np.zeros((C_, H, D)), np.zeros((C_, D)))
    st = State(np.zeros((N, Cprime), np.int32), np.zeros((C_, G), np.int32),
               np.zeros(C_, np.int32), np.zeros(N, np.int32))
    seeds = np.zeros(C_, np.int64)
    check(lib().vmfa_host_initialize(ptr(X), N, D, C_, H, Cprime, G, seed, scale, loading_init,
                                     ptr(floor), ptr(p.pi), ptr(p.mu), ptr(p.lam), ptr(p.psi),
                                     ptr(st.K), ptr(st.g), ptr(st.g_count), ptr(seeds)))
    return p, st, floor, seeds


def train_fixed(sess: Session, seed: int, warmup: int, iters: int, mode: int = KL,
                first_iteration: int = 0):
    """Fixed-count form of train_vmfa (trainer.cpp:111-186): `warmup` E-steps,
    then `iters` main iterations (E-step, statistics, update, precompute,
    truncated F). The global E-step index keys the extra draws."""
    recs = []
    it = first_iteration
    for _ in range(warmup):
        F, J = sess.variational_e_step(seed, it, mode)
        recs.append(dict(warmup=True, F=F, joints=J))
        it += 1
    for _ in range(iters):
        r = sess.iterate(seed, it, mode)
        r["warmup"] = False
        recs.append(r)
        it += 1
    return recs


def check_convergence(f_prev: float, f_curr: float, epsilon: float, literal: bool = False) -> bool:
    """check_convergence (trainer.hpp:76-80): |F - F_prev| < eps |F_prev|;
    literal Eq. 14 uses the signed ratio (F - F_prev) / F_prev < eps."""
    if literal:
        return (f_curr - f_prev) / f_prev < epsilon
    return abs(f_curr - f_prev) < epsilon * abs(f_prev)


@dataclass
class TrainConfig:
    """The training-loop fields of TrainConfig / InitConfig (trainer.hpp:19-37,
    seeding.hpp:18-19) that train_vmfa's loop reads."""
    seed: int = 0
    epsilon: float = 1e-4
    max_iters: int = 500
    mode: int = 0  # KL
    eval_nll_every: int = 0
    literal_eq14: bool = False
    halt_on_max_iters: bool = True
    warmup_epsilon: float = 1e-4
    warmup_max_iters: int = 1000


def train_vmfa(sess: Session, cfg: TrainConfig, testset: Session | None = None) -> dict:
    """train_vmfa's loop (trainer.cpp:111-186) on the device, after the
    caller's initialisation (parameters, floor and state uploaded): warm-up
    E-steps at fixed parameters until check_convergence(warmup_epsilon) or
    MaxIterExceeded, then main iterations (E-step, statistics, update,
    precompute, truncated F) until check_convergence(epsilon); optional exact
    NLL every eval_nll_every iterations (train, and test on a second session
    holding the test rows and the same parameters); final NLL. Returns the
    TrainReport fields (trainer.hpp:39-64) with per-iteration records."""
    import math
    import time

    def nll(s):  # nll_per_point (trainer.cpp:79-85) over one context's rows
        return -s.exact_log_likelihood() / s.N

    def sync_test():
        if testset is not None:
            testset.upload_params(sess.download_params())

    recs, joints = [], 0
    t_start = time.perf_counter()
    empty0 = int((sess.download_params().pi == 0.0).sum())  # count_empty (fixed during warm-up)
    excluded = 0.0
    it_index = 0
    warm, main = 0, 0
    prev = math.nan
    for it in range(cfg.warmup_max_iters):  # trainer.cpp:115-142
        t0 = time.perf_counter()
        F, J = sess.variational_e_step(cfg.seed, it_index, cfg.mode)
        it_index += 1
        warm += 1
        joints += J
        recs.append(dict(t=warm, warmup=True, F=F, joint_evals=joints,
                         wall_ms=(time.perf_counter() - t0) * 1e3, empty_components=empty0))
        if math.isfinite(prev) and check_convergence(prev, F, cfg.warmup_epsilon, cfg.literal_eq14):
            break
        prev = F
        if it + 1 == cfg.warmup_max_iters:
            raise VmfaError(6, "warm-up did not converge")
    prev_f, converged = math.nan, False
    for t in range(1, cfg.max_iters + 1):  # trainer.cpp:147-186
        t0 = time.perf_counter()
        r = sess.iterate(cfg.seed, it_index, cfg.mode)
        it_index += 1
        main += 1
        joints += r["joints"]
        rec = dict(t=t, warmup=False, F=r["F"], F_estep=r["F_estep"], joint_evals=joints,
                   wall_ms=(time.perf_counter() - t0) * 1e3, empty_components=r["empty"],
                   nll_train=math.nan, nll_test=math.nan)
        if cfg.eval_nll_every > 0 and t % cfg.eval_nll_every == 0:
            t1 = time.perf_counter()
            rec["nll_train"] = nll(sess)
            if testset is not None:
                sync_test()
                rec["nll_test"] = nll(testset)
            excluded += time.perf_counter() - t1
        recs.append(rec)
        if math.isfinite(prev_f) and check_convergence(prev_f, r["F"], cfg.epsilon, cfg.literal_eq14):
            converged = True
            break
        prev_f = r["F"]
    if not converged and cfg.halt_on_max_iters:
        raise VmfaError(6, f"training did not converge within {cfg.max_iters} iterations")
    report = dict(algo="vmfa", iterations=recs, warmup_iterations=warm, main_iterations=main,
                  converged=converged, joint_evals=joints,
                  empty_components=recs[-1]["empty_components"],
                  total_wall_ms=(time.perf_counter() - t_start - excluded) * 1e3)
    report["nll_train"] = nll(sess)  # finalize_nll (trainer.cpp:49-56)
    if testset is not None:
        sync_test()
        report["nll_test"] = nll(testset)
    return report


def train_emmfa(sess: Session, cfg: TrainConfig) -> dict:
    """run_emmfa_loop (trainer.cpp:205-260, train_emmfa trainer.hpp:90) on the
    device, after the caller's initialisation: full-posterior EM iterations
    (em_full_step, update_params + precompute, exact log-likelihood F) until
    check_convergence(epsilon) on F, or max_iters; NLL every eval_nll_every
    iterations. Joint evaluations count N*C per em_full_step (the exact-F pass
    is not counted, as the reference's `scratch` counter)."""
    import math
    import time

    recs, joints = [], 0
    t_start = time.perf_counter()
    excluded = 0.0
    prev_f, converged = math.nan, False
    for t in range(1, cfg.max_iters + 1):
        t0 = time.perf_counter()
        _, j = sess.em_full_step()
        joints += j
        sess.update_params()
        f = sess.exact_log_likelihood()
        empty = int((sess.download_params().pi == 0.0).sum())
        rec = dict(t=t, warmup=False, F=f, joint_evals=joints, wall_ms=(time.perf_counter() - t0) * 1e3,
                   empty_components=empty, nll_train=math.nan)
        if cfg.eval_nll_every > 0 and t % cfg.eval_nll_every == 0:
            t1 = time.perf_counter()
            rec["nll_train"] = -f / sess.N  # nll_per_point (trainer.cpp:79-85) of the same parameters
            excluded += time.perf_counter() - t1
        recs.append(rec)
        if math.isfinite(prev_f) and check_convergence(prev_f, f, cfg.epsilon, cfg.literal_eq14):
            converged = True
            break
        prev_f = f
    if not converged and cfg.halt_on_max_iters:  # run_emmfa_loop, use_eq14 path (trainer.cpp:262-266)
        raise VmfaError(6, f"full EM did not converge within {cfg.max_iters} iterations")
    report = dict(algo="emmfa", iterations=recs, warmup_iterations=0, main_iterations=len(recs),
                  converged=converged, joint_evals=joints, empty_components=recs[-1]["empty_components"],
                  total_wall_ms=(time.perf_counter() - t_start - excluded) * 1e3)
    report["nll_train"] = -sess.exact_log_likelihood() / sess.N
    return report


# ---- on-disk containers (io.hpp:12-23; host only) -----------------------------
def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def save_dataset(path, X: np.ndarray) -> None:
    """MFAD (io.cpp:91-104): bit-exact f32 rows."""
    X = _c(X, np.float32)
    check(lib().vmfa_save_dataset(_path(path), ptr(X), X.shape[0], X.shape[1]))


def dataset_info(path) -> tuple[int, int]:
    n, d = C.c_int64(), C.c_int()
    check(lib().vmfa_dataset_info(_path(path), C.byref(n), C.byref(d)))
    return n.value, d.value


def load_dataset(path, row_begin: int = 0, rows: int | None = None) -> np.ndarray:
    """MFAD (io.cpp:106-125); a row range reads one shard."""
    n, d = dataset_info(path)
    rows = n - row_begin if rows is None else rows
    X = np.empty((rows, d), np.float32)
    check(lib().vmfa_load_dataset(_path(path), row_begin, rows, d, ptr(X)))
    return X


def save_checkpoint(path, p: Params) -> None:
    """MFAM (io.cpp:127-149), MfaParams::validate first."""
    C_, D = p.mu.shape
    H = p.lam.shape[1]
    check(lib().vmfa_save_checkpoint(_path(path), C_, D, H, ptr(_c(p.pi, np.float64)), ptr(_c(p.mu, np.float64)),
                                     ptr(_c(p.lam, np.float64)), ptr(_c(p.psi, np.float64))))


def load_checkpoint(path) -> Params:
    """MFAM (io.cpp:151-179)."""
    c, d, h = C.c_int(), C.c_int(), C.c_int()
    check(lib().vmfa_checkpoint_info(_path(path), C.byref(c), C.byref(d), C.byref(h)))
    C_, D, H = c.value, d.value, h.value
    p = Params(np.empty(C_), np.empty((C_, D)), np.empty((C_, H, D)), np.empty((C_, D)))
    check(lib().vmfa_load_checkpoint(_path(path), C_, D, H, ptr(p.pi), ptr(p.mu), ptr(p.lam), ptr(p.psi)))
    return p


def save_state(path, st: State) -> None:
    """MFAK sidecar: K, g, g_count (exact resume)."""
    K = _c(st.K, np.int32)
    g = _c(st.g, np.int32)
    check(lib().vmfa_save_state(_path(path), K.shape[0], K.shape[1], g.shape[0], g.shape[1], ptr(K), ptr(g),
                                ptr(_c(st.g_count, np.int32))))


def load_state(path, row_begin: int = 0, rows: int | None = None) -> State:
    n, cp, c, gg = C.c_int64(), C.c_int(), C.c_int(), C.c_int()
    check(lib().vmfa_state_info(_path(path), C.byref(n), C.byref(cp), C.byref(c), C.byref(gg)))
    rows = n.value - row_begin if rows is None else rows
    st = State(np.empty((rows, cp.value), np.int32), np.empty((c.value, gg.value), np.int32),
               np.empty(c.value, np.int32))
    check(lib().vmfa_load_state(_path(path), row_begin, rows, cp.value, c.value, gg.value, ptr(st.K), ptr(st.g),
                                ptr(st.g_count)))
    return st


def write_report_jsonl(report: dict, out) -> None:
    """TrainReport as JSON lines (SPEC.md 'External Interfaces'): one object
    per iteration, then a final summary object. `out`: path or text stream;
    NaN NLLs (not evaluated) are written as null."""
    import json
    import math

    def clean(v):
        return None if isinstance(v, float) and math.isnan(v) else v

    f = open(out, "w") if isinstance(out, (str, os.PathLike)) else out
    try:
        for r in report["iterations"]:
            f.write(json.dumps({k: clean(v) for k, v in r.items()}) + "\n")
        summary = {k: clean(v) for k, v in report.items() if k != "iterations"}
        summary["summary"] = True
        f.write(json.dumps(summary) + "\n")
    finally:
        if f is not out:
            f.close()


__all__ = ["Params", "State", "Stats", "Session", "CONFIGS", "synth_spec", "gen_synthetic",
           "initialize", "train_fixed", "train_vmfa", "TrainConfig", "check_convergence", "write_report_jsonl",
           "save_dataset", "load_dataset", "dataset_info", "save_checkpoint", "load_checkpoint", "save_state",
           "load_state",
           "device_available", "VmfaError", "KL", "EUCLID"]
