"""CPU tests of the product library's host side and its C-ABI surface:
  * libvmfa_b200.so loads without a GPU and exports every symbol declared in
    include/vmfa_b200.h;
  * error behaviour without a device (NoDevice, mapped like the reference's
    exception types, errors.hpp:9-62) and argument validation;
  * the host-side initialisation (trainer.cpp:32-47, 107-109) is bit-identical
    to the oracle's restatement; the synthetic generators are deterministic
    and shard-consistent.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "vmfa_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(vmfa_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("vmfa_ctx_create", "vmfa_estep", "vmfa_iterate", "vmfa_accumulate_suffstats",
                 "vmfa_update_params", "vmfa_precompute", "vmfa_truncated_free_energy",
                 "vmfa_exchange_buffer", "vmfa_host_initialize", "vmfa_gen_synthetic",
                 "vmfa_exact_log_likelihood", "vmfa_em_full_step", "vmfa_afkmc2_seed",
                 "vmfa_cooc_sparse", "vmfa_cooc_local_list", "vmfa_cooc_select"):
        assert must in names


def test_library_exports_every_declared_symbol(vmfa):
    from paper_2501_12299_b200 import abi
    lib = C.CDLL(abi.library_path())
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert abi.lib().vmfa_abi_version() == 1


def test_no_device_is_reported_not_faked(vmfa):
    from paper_2501_12299_b200 import abi
    if vmfa.device_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(abi.VmfaError) as ei:
        vmfa.Session(4, 3, 1, 2, 2, np.zeros((10, 3), np.float32))
    assert ei.value.code == 101  # VMFA_ERR_NO_DEVICE: no CPU fallback exists


def test_invalid_arguments_map_to_invalid_argument(vmfa):
    from paper_2501_12299_b200 import abi
    h = C.c_void_p()
    # C' > C and H > D are std::invalid_argument in the reference (trainer.cpp:60-77)
    assert abi.lib().vmfa_ctx_create(C.byref(h), 0, 4, 3, 1, 5, 2, 10, 0, 10, None) == 1
    assert abi.lib().vmfa_ctx_create(C.byref(h), 0, 4, 3, 4, 2, 2, 10, 0, 10, None) == 1
    assert b"invalid sizes" in abi.lib().vmfa_last_error()


def test_unsupported_shapes_are_rejected_before_any_device_work(vmfa):
    from paper_2501_12299_b200 import abi
    h = C.c_void_p()
    # G > 64: the g-selection kernels hold the picks in 64-entry arrays; C'=1 keeps C'G+1 <= 256
    assert abi.lib().vmfa_ctx_create(C.byref(h), 0, 200, 8, 2, 1, 65, 100, 0, 100, None) == 102
    assert b"G <= 64" in abi.lib().vmfa_last_error()
    assert abi.lib().vmfa_ctx_create(C.byref(h), 0, 200, 8, 2, 9, 5, 100, 0, 100, None) == 102


def test_host_initialize_matches_oracle(oracle, vmfa):
    X = vmfa.gen_synthetic(vmfa.synth_spec(1, N=3000))
    for li, sc in ((1, 0.1), (0, 1.0)):
        p, st, floor, seeds = vmfa.initialize(X, 50, 4, 3, 5, seed=7, scale=sc, loading_init=li)
        po, sto, flo, so = oracle.initialize(X, 50, 4, 3, 5, seed=7, scale=sc, loading_init=li)
        assert np.array_equal(seeds, so)
        assert np.array_equal(st.K, sto.K) and np.array_equal(st.g, sto.g)
        assert np.array_equal(st.g_count, sto.g_count)
        np.testing.assert_array_equal(p.mu, po.mu)
        np.testing.assert_array_equal(p.lam, po.lam)
        np.testing.assert_allclose(p.psi, po.psi, rtol=1e-13)
        np.testing.assert_allclose(floor, flo, rtol=1e-13)


def test_synthetic_rows_identical_in_oracle_build(oracle, vmfa):
    """The BASELINE generator compiled into the oracle (reference arm) and into
    the product (GPU arm) gives bit-identical rows, and both config tables agree."""
    for cfg in (1, 2, 3, 4, 5):
        assert oracle.CONFIGS[cfg] == {k: dict(v) for k, v in vmfa.CONFIGS[cfg].items()}
        over = {"C_true": 300} if cfg == 5 else {}
        a = vmfa.gen_synthetic(vmfa.synth_spec(cfg, N=5000, **over), 1000, 1400)
        b = oracle.gen_synthetic(oracle.synth_spec(cfg, N=5000, **over), 1000, 1400)
        assert a.tobytes() == b.tobytes(), cfg


def _fill_distinct_numpy(draws, C, want, preset):
    """seeding.cpp:187-203 literally: a C-sized buffer 0..C-1, the preset swap,
    j = i + uniform_int(C - i) swaps (uniform_int = mulhi(next_u64, bound),
    rng.hpp:55-60), then the first `want` entries sorted."""
    buf = np.arange(C)
    start = 0
    if preset >= 0:
        buf[0], buf[preset] = buf[preset], buf[0]
        start = 1
    for i in range(start, want):
        u = int(next(draws))
        j = i + ((u * (C - i)) >> 64)
        buf[i], buf[j] = buf[j], buf[i]
    return np.sort(buf[:want])


def test_init_varstate_pinned_to_dense_fill_distinct(oracle, vmfa):
    """init_varstate (seeding.cpp:207-233) three ways: a numpy restatement of
    the dense fill_distinct over the golden-pinned stream (orc_rng_u64, checked
    bit-exactly against the reference's rng.hpp in test_oracle_pins), the
    oracle's dense C++ restatement, and the product's sparse swap map."""
    X = vmfa.gen_synthetic(vmfa.synth_spec(1, N=700))
    C, H, Cp, G, seed = 37, 2, 4, 6, 9
    p, st, floor, seeds = vmfa.initialize(X, C, H, Cp, G, seed=seed)
    so = oracle.init_varstate(X.shape[0], C, Cp, G, seeds, oracle.hash_combine(seed, oracle.STATE_SALT))
    n_draws = X.shape[0] * Cp + C * G
    draws = iter(oracle.rng_u64(oracle.hash_combine(seed, oracle.STATE_SALT), n_draws))
    seed_of = {int(n): c for c, n in enumerate(seeds)}
    K = np.stack([_fill_distinct_numpy(draws, C, Cp, seed_of.get(n, -1)) for n in range(X.shape[0])])
    g = np.stack([_fill_distinct_numpy(draws, C, G, c) for c in range(C)])
    assert np.array_equal(K, so.K) and np.array_equal(K, st.K)
    assert np.array_equal(g, so.g) and np.array_equal(g, st.g)


def test_sharded_initialize_single_rank_matches(vmfa):
    from paper_2501_12299_b200.sharded import initialize_sharded
    X = vmfa.gen_synthetic(vmfa.synth_spec(2, N=3000))
    p, st, floor, seeds = vmfa.initialize(X, 200, 8, 5, 10, seed=4)
    p2, st2, floor2, seeds2 = initialize_sharded(X, 0, X.shape[0], 200, 8, 5, 10, seed=4)
    assert np.array_equal(seeds, seeds2) and np.array_equal(st.K, st2.K) and np.array_equal(st.g, st2.g)
    for f in ("pi", "mu", "lam", "psi"):
        assert np.array_equal(getattr(p, f), getattr(p2, f)), f
    assert np.array_equal(floor, floor2)


def test_degenerate_data_is_reported(vmfa):
    from paper_2501_12299_b200.sharded import initialize_sharded
    X = np.repeat(vmfa.gen_synthetic(vmfa.synth_spec(1, N=50), 0, 5), 10, axis=0)
    with pytest.raises(vmfa.VmfaError, match="DegenerateData"):
        vmfa.initialize(X, 8, 2, 2, 3)
    with pytest.raises(vmfa.VmfaError, match="DegenerateData"):
        initialize_sharded(X, 0, X.shape[0], 8, 2, 2, 3)
    # -0.0 and +0.0 are one value to the reference's row compare (seeding.cpp:26, :140)
    X = vmfa.gen_synthetic(vmfa.synth_spec(1, N=50), 0, 12)
    X[1, 0] = 0.0
    X[5] = X[1]
    X[5, 0] = -0.0
    for impl in (lambda C_: vmfa.initialize(X, C_, 2, 2, 3),
                 lambda C_: initialize_sharded(X, 0, X.shape[0], C_, 2, 2, 3)):
        with pytest.raises(vmfa.VmfaError, match="DegenerateData"):
            impl(12)
        seeds = impl(11)[3]
        assert len(set(seeds.tolist()) & {1, 5}) == 1 and len(set(seeds.tolist())) == 11


def test_init_varstate_invariants(vmfa):
    X = vmfa.gen_synthetic(vmfa.synth_spec(2, N=5000))
    p, st, floor, seeds = vmfa.initialize(X, 300, 8, 5, 10, seed=3)
    assert np.all(np.diff(st.K, axis=1) > 0) and st.K.min() >= 0 and st.K.max() < 300
    for c in range(300):
        row = st.g[c, :st.g_count[c]]
        assert c in row and np.all(np.diff(row) > 0)
    # seed rows carry their own component (seeding.cpp:215-218)
    for c, n in enumerate(seeds):
        assert c in st.K[n]
    assert np.all(p.pi == 1.0 / 300)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generators_deterministic_and_shardable(vmfa, cfg):
    # config 5's 50 000 ground-truth fields are reduced to 500 here (CPU time)
    sp = vmfa.synth_spec(cfg, N=600, **({"C_true": 500} if cfg == 5 else {}))
    a = vmfa.gen_synthetic(sp)
    b = vmfa.gen_synthetic(sp, threads=1)
    assert np.array_equal(a, b)
    assert np.array_equal(vmfa.gen_synthetic(sp, 200, 400), a[200:400])
    assert np.isfinite(a).all() and a.shape == (600, sp.D)
    if vmfa.CONFIGS[cfg]["truth"]["kind"] == 1:
        assert a.min() >= 0.0 and a.max() <= 1.0  # clipped image-like fields


def test_error_codes_cover_the_reference_exceptions():
    src = open(HEADER).read()
    for name in ("CholeskyFailure", "EmptyKSet", "InsufficientCandidates", "SingularEc",
                 "MaxIterExceeded", "TargetUnreachable", "DegenerateData", "BadMagic",
                 "TruncatedFile", "UnsupportedVersion"):
        assert name in src


def build_facade(tmp_path):
    import subprocess
    exe = tmp_path / "facade_train"
    lib_dir = os.path.join(ROOT, "paper_2501_12299_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_train.cpp"), "-L", lib_dir,
                    "-lvmfa_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_mirror_compiles_and_reports_no_device(vmfa, tmp_path):
    import subprocess
    exe = build_facade(tmp_path)
    if vmfa.device_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([str(exe), "200"], capture_output=True, text=True)
    assert r.returncode == 3 and "no sm_100" in r.stderr


def test_report_jsonl_and_convergence_rule():
    # SPEC.md 'External Interfaces': one JSON object per iteration + a final
    # summary; check_convergence (trainer.hpp:76-80) in both readings
    import io
    import json
    import math
    from paper_2501_12299_b200 import vmfa as V
    assert V.check_convergence(-100.0, -100.005, 1e-4)
    assert not V.check_convergence(-100.0, -100.02, 1e-4)
    assert V.check_convergence(-100.0, -99.0, 1e-4, literal=True)  # any improvement fires
    rep = dict(algo="vmfa", iterations=[dict(t=1, warmup=True, F=-5.0, nll_train=math.nan),
                                        dict(t=1, warmup=False, F=-4.0, nll_train=2.5)],
               warmup_iterations=1, main_iterations=1, converged=True, joint_evals=10, nll_train=2.4)
    buf = io.StringIO()
    V.write_report_jsonl(rep, buf)
    lines = [json.loads(l) for l in buf.getvalue().splitlines()]
    assert len(lines) == 3 and lines[0]["nll_train"] is None and lines[1]["nll_train"] == 2.5
    assert lines[2]["summary"] and lines[2]["converged"] and "iterations" not in lines[2]


def build_fit_fa(tmp_path):
    import subprocess
    exe = tmp_path / "fit_fa"
    lib_dir = os.path.join(ROOT, "paper_2501_12299_b200", "_lib")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "fit_fa.cpp"), "-L", lib_dir,
                    "-lvmfa_b200", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_fit_fa_program_compiles(vmfa, tmp_path):
    assert build_fit_fa(tmp_path).exists()
