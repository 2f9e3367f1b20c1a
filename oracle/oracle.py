"""ctypes wrapper over the fp64 CPU oracle (oracle/vmfa_oracle.cpp).

TEST INFRASTRUCTURE ONLY. Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs -- never from the product
package (paper_2501_12299_b200/). Every function mirrors the reference free
function named in its docstring (paths relative to /root/reference/).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libvmfa_oracle.so")
_lib = None

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")

STATUS_NAMES = {
    0: "OK", 1: "InvalidArgument", 2: "CholeskyFailure", 3: "EmptyKSet",
    4: "InsufficientCandidates", 5: "SingularEc", 6: "MaxIterExceeded",
    7: "TargetUnreachable", 8: "DegenerateData",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {what}")


def build() -> str:
    """Compile the oracle with its Makefile (g++ only, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        u64, i64, i32, f64 = C.c_uint64, C.c_int64, C.c_int, C.c_double
        L.orc_hash_combine.restype = u64
        L.orc_hash_combine.argtypes = [u64, u64]
        L.orc_hash3.restype = u64
        L.orc_hash3.argtypes = [u64, u64, u64]
        L.orc_uniform_component.restype = i32
        L.orc_uniform_component.argtypes = [u64, u64, u64, i32]
        L.orc_rng_u64.argtypes = [u64, i32, u64p]
        L.orc_rng_ops.argtypes = [u64, i32, i32p, i64p, f64p]
        L.orc_log_sum_exp.restype = f64
        L.orc_log_sum_exp.argtypes = [f64p, i32]
        L.orc_per_dimension_variance.argtypes = [f32p, i64, i32, f64p]
        L.orc_variance_floor.argtypes = [f32p, i64, i32, f64p]
        L.orc_precompute.argtypes = [i32, i32, i32, f64p, f64p, f64p, f64p, f64p, f64p, f64p,
                                     f64p, f64p, f64p, f64p, C.POINTER(C.c_int)]
        L.orc_log_joint.restype = f64
        L.orc_log_joint.argtypes = [i32, i32, f64p, f64p, f64p, f64, f64, f64p, f32p]
        L.orc_estep.argtypes = [i64, i32, i32, i32, i32, i32, f32p, f64p, f64p, f64p, f64p, f64p,
                                f64p, f64p, f64p, f64p, i32p, i32p, i32p, i32p, u64, u64, i32, i32,
                                i32p, i32p, f64p, f64p, C.POINTER(C.c_double),
                                C.POINTER(C.c_uint64), i64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.POINTER(C.c_int64), u64]
        L.orc_suffstats.argtypes = [i64, i32, i32, i32, i32, f32p, f64p, f64p, f64p, i32p, f64p,
                                    i32, f64p, f64p, f64p, f64p]
        L.orc_update_params.argtypes = [i32, i32, i32, i64, f64p, f64p, f64p, f64p, f64p, f64p,
                                        f64p, f64p, f64p, f64p, f64p, f64p, f64p,
                                        C.POINTER(C.c_int)]
        L.orc_truncated_F.argtypes = [i64, i32, i32, i32, i32, f32p, f64p, f64p, f64p, f64p, f64p,
                                      f64p, f64p, f64p, i32p, i32, C.POINTER(C.c_double),
                                      C.c_void_p]
        L.orc_exact_ll.argtypes = [i64, i32, i32, i32, f32p, f64p, f64p, f64p, f64p, f64p, f64p,
                                   f64p, f64p, i32, C.POINTER(C.c_double)]
        L.orc_random_points_seed.argtypes = [f32p, i64, i32, i32, u64, i64p, u64p]
        L.orc_afkmc2.argtypes = [f32p, i64, i32, i32, i32, u64, i64p, u64p, u64p]
        L.orc_init_params.argtypes = [f32p, i64, i32, i32, i32, i64p, u64p, f64, i32, f64p, f64p,
                                      f64p, f64p, f64p]
        L.orc_init_varstate.argtypes = [i64, i32, i32, i32, i64p, i32, u64, i32p, i32p, i32p]
        L.orc_gen_synthetic.argtypes = [C.c_void_p, i64, i64, C.c_void_p, C.c_void_p, i32]
        _lib = L
    return _lib


def _check(code: int, what: str = ""):
    if code != 0:
        raise OracleError(code, what)


# ------------------------------------------------------------------ containers
@dataclass
class Params:
    """MfaParams (model.hpp:19-32): pi (C), mu (C,D), lam (C,H,D) -- i.e. the
    reference's per-component column-major D x H block --, psi (C,D)."""
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
class Caches:
    """ComponentCache (model.hpp:37-45) for all C components."""
    U: np.ndarray      # (C,H,D)  = D x H col-major blocks
    Lmat: np.ndarray   # (C,H,H)  col-major
    V: np.ndarray      # (C,D,H)  = H x D col-major blocks
    Sz: np.ndarray     # (C,H,H)
    inv_psi: np.ndarray  # (C,D)
    logdet: np.ndarray   # (C,)
    log_pi: np.ndarray   # (C,)


@dataclass
class State:
    """VarState (estep.hpp:17-29): K (N,C'), g (C,G) -1 padded, g_count (C,), labels (N,)."""
    K: np.ndarray
    g: np.ndarray
    g_count: np.ndarray
    labels: np.ndarray = field(default=None)

    def copy(self):
        return State(self.K.copy(), self.g.copy(), self.g_count.copy(),
                     None if self.labels is None else self.labels.copy())


@dataclass
class EStep:
    """EStepResult (estep.hpp:72-78) plus the block-3 accumulator dump."""
    count: np.ndarray
    idx: np.ndarray
    lj: np.ndarray
    resp: np.ndarray
    F: float
    joints: int
    dist: tuple | None = None  # (c, ct, sum, count) arrays, (c, ct) ascending


@dataclass
class Stats:
    """SuffStats (mstep.hpp:14-22)."""
    Nc: np.ndarray   # (C,)
    Y: np.ndarray    # (C,H+1,D)  = D x (H+1) col-major blocks
    E: np.ndarray    # (C,H+1,H+1) col-major
    sq: np.ndarray   # (C,D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------ RNG
def hash_combine(a: int, b: int) -> int:
    return int(lib().orc_hash_combine(a, b))


def hash3(a: int, b: int, c: int) -> int:
    return int(lib().orc_hash3(a, b, c))


def uniform_component(seed: int, iteration: int, n: int, C_: int) -> int:
    return int(lib().orc_uniform_component(seed, iteration, n, C_))


def rng_u64(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    lib().orc_rng_u64(seed, n, out)
    return out


def rng_ops(seed: int, ops, bounds=None) -> np.ndarray:
    ops = np.asarray(ops, np.int32)
    b = np.zeros(len(ops), np.int64) if bounds is None else np.asarray(bounds, np.int64)
    out = np.zeros(len(ops), np.float64)
    lib().orc_rng_ops(seed, len(ops), ops, b, out)
    return out


def log_sum_exp(v) -> float:
    v = _f64(v)
    return float(lib().orc_log_sum_exp(v, len(v)))


# ------------------------------------------------------------------ data / model
def per_dimension_variance(X):
    X = _f32(X)
    out = np.zeros(X.shape[1])
    lib().orc_per_dimension_variance(X, X.shape[0], X.shape[1], out)
    return out


def variance_floor(X):
    X = _f32(X)
    out = np.zeros(X.shape[1])
    lib().orc_variance_floor(X, X.shape[0], X.shape[1], out)
    return out


def precompute_all(p: Params) -> Caches:
    """precompute_all / precompute_component (model.cpp:43-79)."""
    C_, D, H = p.C, p.D, p.H
    k = Caches(np.zeros((C_, H, D)), np.zeros((C_, H, H)), np.zeros((C_, D, H)),
               np.zeros((C_, H, H)), np.zeros((C_, D)), np.zeros(C_), np.zeros(C_))
    bad = C.c_int(-1)
    code = lib().orc_precompute(C_, D, H, _f64(p.pi), _f64(p.mu), _f64(p.lam), _f64(p.psi),
                                k.U, k.Lmat, k.V, k.Sz, k.inv_psi, k.logdet, k.log_pi,
                                C.byref(bad))
    _check(code, f"component {bad.value}")
    return k


def log_joint(k: Caches, mu: np.ndarray, c: int, x) -> float:
    """log_joint (model.cpp:81-95) for component c at row x."""
    D, H = mu.shape[1], k.U.shape[1]
    return float(lib().orc_log_joint(D, H, _f64(k.U[c]), _f64(k.V[c]), _f64(k.inv_psi[c]),
                                     float(k.logdet[c]), float(k.log_pi[c]), _f64(mu[c]),
                                     _f32(x)))


def variational_e_step(X, p: Params, k: Caches, st: State, seed: int, iteration: int,
                       mode: int = 0, threads: int = 1, dump_distances: bool = False,
                       n_offset: int = 0) -> EStep:
    """variational_e_step (estep.cpp:230-336). Updates st in place (K, g, labels)."""
    X = _f32(X)
    N, D = X.shape
    C_, Cp, G = p.C, st.K.shape[1], st.g.shape[1]
    H = p.H
    stride = min(Cp * G + 1, C_)
    if st.labels is None or st.labels.shape != (N,):
        st.labels = np.zeros(N, np.int32)
    cnt = np.zeros(N, np.int32)
    idx = np.zeros(N * stride, np.int32)
    lj = np.zeros(N * stride, np.float64)
    resp = np.zeros(N * Cp, np.float64)
    F = C.c_double()
    J = C.c_uint64()
    dn = C.c_int64(0)
    cap = 0
    bufs = [None] * 4
    if dump_distances:
        cap = N * stride
        bufs = [np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(cap, np.float64),
                np.zeros(cap, np.int64)]
    ptr = [None if b is None else b.ctypes.data_as(C.c_void_p) for b in bufs]
    code = lib().orc_estep(N, D, H, C_, Cp, G, X, _f64(p.pi), _f64(p.mu), k.U, k.Lmat, k.V,
                           k.Sz, k.inv_psi, k.logdet, k.log_pi, st.K, st.g, st.g_count,
                           st.labels, seed, iteration, mode, threads, cnt, idx, lj, resp,
                           C.byref(F), C.byref(J), cap, ptr[0], ptr[1], ptr[2], ptr[3],
                           C.byref(dn), n_offset)
    _check(code, "variational_e_step")
    dist = None
    if dump_distances:
        m = dn.value
        dist = tuple(b[:m].copy() for b in bufs)
    return EStep(cnt, idx.reshape(N, stride), lj.reshape(N, stride), resp.reshape(N, Cp),
                 F.value, J.value, dist)


def accumulate_suffstats(X, p: Params, k: Caches, K, resp, threads: int = 1) -> Stats:
    """accumulate_suffstats (mstep.cpp:71-101)."""
    X = _f32(X)
    N, D = X.shape
    C_, H, Cp = p.C, p.H, K.shape[1]
    s = Stats(np.zeros(C_), np.zeros((C_, H + 1, D)), np.zeros((C_, H + 1, H + 1)),
              np.zeros((C_, D)))
    code = lib().orc_suffstats(N, D, H, C_, Cp, X, _f64(p.mu), k.V, k.Sz, _i32(K), _f64(resp),
                               threads, s.Nc, s.Y, s.E, s.sq)
    _check(code, "accumulate_suffstats")
    return s


def update_params(s: Stats, N: int, prev: Params, floor) -> Params:
    """update_params (mstep.cpp:103-162)."""
    C_, D, H = prev.C, prev.D, prev.H
    out = Params(np.zeros(C_), np.zeros((C_, D)), np.zeros((C_, H, D)), np.zeros((C_, D)))
    bad = C.c_int(-1)
    code = lib().orc_update_params(C_, D, H, N, _f64(s.Nc), _f64(s.Y), _f64(s.E), _f64(s.sq),
                                   _f64(floor), _f64(prev.pi), _f64(prev.mu), _f64(prev.lam),
                                   _f64(prev.psi), out.pi, out.mu, out.lam, out.psi,
                                   C.byref(bad))
    _check(code, f"component {bad.value}")
    return out


def truncated_free_energy(X, p: Params, k: Caches, K, threads: int = 1, return_lj=False):
    """truncated_free_energy (model.cpp:150-159)."""
    X = _f32(X)
    N, D = X.shape
    Cp = K.shape[1]
    F = C.c_double()
    lj = np.zeros((N, Cp)) if return_lj else None
    code = lib().orc_truncated_F(N, D, p.H, p.C, Cp, X, _f64(p.mu), k.U, k.Lmat, k.V, k.Sz,
                                 k.inv_psi, k.logdet, k.log_pi, _i32(K), threads, C.byref(F),
                                 None if lj is None else lj.ctypes.data_as(C.c_void_p))
    _check(code, "truncated_free_energy")
    return (F.value, lj) if return_lj else F.value


def exact_log_likelihood(X, p: Params, k: Caches, threads: int = 1) -> float:
    """exact_log_likelihood (model.cpp:139-148)."""
    X = _f32(X)
    N, D = X.shape
    F = C.c_double()
    code = lib().orc_exact_ll(N, D, p.H, p.C, X, _f64(p.mu), k.U, k.Lmat, k.V, k.Sz, k.inv_psi,
                              k.logdet, k.log_pi, threads, C.byref(F))
    _check(code)
    return F.value


def em_full_step(X, p: Params, k: Caches, threads: int = 1):
    """em_full_step (mstep.cpp:164-208): log_joint of every (n, c)
    (model.cpp:81-95, via orc_truncated_F with K = all components), per-row
    log_sum_exp (numerics.hpp:15-22), q = exp(l - lse) over all C and
    accumulate_point for every pair (the orc_suffstats restatement of
    mstep.cpp:47-67 with K = all components, merged in worker order).
    Returns (stats, ll, joints = N*C)."""
    X = _f32(X)
    N = X.shape[0]
    K = np.tile(np.arange(p.C, dtype=np.int32), (N, 1))
    ll, lj = truncated_free_energy(X, p, k, K, threads=threads, return_lj=True)
    lse = np.array([log_sum_exp(row) for row in lj])
    resp = np.exp(lj - lse[:, None])
    stats = accumulate_suffstats(X, p, k, K, resp, threads=threads)
    return stats, ll, N * p.C


# ------------------------------------------------------------------ benchmark inputs
class SynthSpec(C.Structure):
    """vmfa_synth_spec (include/vmfa_b200.h): one BASELINE config's generator."""
    _fields_ = [("kind", C.c_int), ("n_total", C.c_int64), ("D", C.c_int), ("C_true", C.c_int),
                ("H_true", C.c_int), ("dirichlet", C.c_int), ("mu_std", C.c_double),
                ("lam_std", C.c_double), ("psi_lo", C.c_double), ("psi_hi", C.c_double),
                ("noise_std", C.c_double), ("img_w", C.c_int), ("img_h", C.c_int),
                ("img_c", C.c_int), ("blur_sigma", C.c_double), ("data_seed", C.c_uint64)]


# BASELINE.json configs: truth generator + fitted model. The
# product's table (paper_2501_12299_b200/vmfa.py CONFIGS) is asserted equal
# in tests/test_abi_host.py; the oracle keeps its own so the reference arm
# never imports the product.
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
    for k in ("D", "C_true", "H_true"):
        setattr(sp, k, t[k])
    for k in ("dirichlet", "img_w", "img_h", "img_c"):
        setattr(sp, k, t.get(k, 0))
    for k in ("mu_std", "lam_std", "psi_lo", "psi_hi", "noise_std", "blur_sigma"):
        setattr(sp, k, t.get(k, 0.0))
    sp.data_seed = data_seed
    return sp


def gen_synthetic(spec: SynthSpec, row_begin: int = 0, row_end: int | None = None, threads: int = 0):
    """Rows [row_begin, row_end) of a BASELINE config: the generator source
    shared with the product (csrc/host/vmfa_synth.cpp), compiled into this
    library -- bit-identical rows, no product library loaded."""
    row_end = spec.n_total if row_end is None else row_end
    X = np.empty((row_end - row_begin, spec.D), np.float32)
    _check(lib().orc_gen_synthetic(C.byref(spec), row_begin, row_end, X.ctypes.data_as(C.c_void_p), None,
                                   threads or (os.cpu_count() or 1)), "gen_synthetic")
    return X


# ------------------------------------------------------------------ init (trainer.cpp:32-47, 107)
INIT_SALT = 0x1217F01D   # trainer.cpp:36
STATE_SALT = 0x7A57A7E5  # trainer.cpp:107


def random_points_seed(X, C_: int, stream_seed: int):
    """random_points_seed (seeding.cpp:123-149); returns (seeds, stream state after)."""
    X = _f32(X)
    seeds = np.zeros(C_, np.int64)
    state = np.zeros(4, np.uint64)
    _check(lib().orc_random_points_seed(X, X.shape[0], X.shape[1], C_, stream_seed, seeds, state))
    return seeds, state


def afkmc2_seed(X, C_: int, chain_length: int, stream_seed: int):
    """afkmc2_seed (seeding.cpp:60-121); returns (seeds, stream state after,
    squared_distance calls)."""
    X = _f32(X)
    seeds = np.zeros(C_, np.int64)
    state = np.zeros(4, np.uint64)
    cnt = np.zeros(1, np.uint64)
    _check(lib().orc_afkmc2(X, X.shape[0], X.shape[1], C_, chain_length, stream_seed, seeds, state, cnt))
    return seeds, state, int(cnt[0])


def init_params(X, C_: int, H: int, seeds, stream_state, floor, scale: float = 1.0,
                loading_init: int = 0) -> Params:
    """init_params (seeding.cpp:151-181). loading_init=1 draws N(0, scale^2)."""
    X = _f32(X)
    N, D = X.shape
    p = Params(np.zeros(C_), np.zeros((C_, D)), np.zeros((C_, H, D)), np.zeros((C_, D)))
    _check(lib().orc_init_params(X, N, D, C_, H, np.ascontiguousarray(seeds, np.int64),
                                 np.ascontiguousarray(stream_state, np.uint64), scale,
                                 loading_init, _f64(floor), p.pi, p.mu, p.lam, p.psi))
    return p


def init_varstate(N: int, C_: int, Cp: int, G: int, seed_rows, stream_seed: int) -> State:
    """init_varstate (seeding.cpp:207-233)."""
    K = np.zeros((N, Cp), np.int32)
    g = np.zeros((C_, G), np.int32)
    gc = np.zeros(C_, np.int32)
    sr = np.ascontiguousarray(seed_rows, np.int64)
    _check(lib().orc_init_varstate(N, C_, Cp, G, sr, len(sr), stream_seed, K, g, gc))
    return State(K, g, gc, np.zeros(N, np.int32))


def initialize(X, C_: int, H: int, Cp: int, G: int, seed: int = 0, scale: float = 1.0,
               loading_init: int = 0):
    """trainer.cpp:32-47 + :107-109 with the random-points seeding."""
    floor = variance_floor(X)
    seeds, st = random_points_seed(X, C_, hash_combine(seed, INIT_SALT))
    p = init_params(X, C_, H, seeds, st, floor, scale, loading_init)
    state = init_varstate(np.asarray(X).shape[0], C_, Cp, G, seeds, hash_combine(seed, STATE_SALT))
    return p, state, floor, seeds


def train_fixed(X, p: Params, st: State, floor, seed: int, warmup: int, iters: int,
                mode: int = 0, threads: int = 1):
    """train_vmfa main structure (trainer.cpp:111-186) with FIXED warm-up and
    main-iteration counts. Returns (params, state, records)."""
    recs = []
    k = precompute_all(p)
    it = 0
    for _ in range(warmup):
        e = variational_e_step(X, p, k, st, seed, it, mode, threads)
        recs.append(dict(warmup=True, F=e.F, joints=e.joints))
        it += 1
    for _ in range(iters):
        e = variational_e_step(X, p, k, st, seed, it, mode, threads)
        it += 1
        s = accumulate_suffstats(X, p, k, st.K, e.resp, threads)
        p = update_params(s, np.asarray(X).shape[0], p, floor)
        k = precompute_all(p)
        F = truncated_free_energy(X, p, k, st.K, threads)
        recs.append(dict(warmup=False, F_estep=e.F, F=F, joints=e.joints,
                         empty=int((p.pi == 0.0).sum())))
    return p, st, recs
