"""On-disk containers: MFAD dataset and MFAM checkpoint
byte layouts as io.cpp:91-179 writes them (rebuilt here with struct.pack from
the reference's field list), bit-exact round trips, shard-range reads, the
MFAK state sidecar, and the reference's error types (BadMagic, TruncatedFile,
UnsupportedVersion, invalid_argument from MfaParams::validate). Host only."""
import struct

import numpy as np
import pytest

from paper_2501_12299_b200 import vmfa as V


def _params(C, D, H, seed=0):
    rng = np.random.default_rng(seed)
    pi = rng.random(C)
    pi /= pi.sum()
    pi[-1] = 1.0 - pi[:-1].sum()
    return V.Params(pi, rng.normal(size=(C, D)), rng.normal(size=(C, H, D)), rng.random((C, D)) + 0.1)


def test_mfad_layout_and_round_trip(tmp_path):
    X = np.random.default_rng(1).normal(size=(37, 5)).astype(np.float32)
    X[3, 2] = np.float32(-0.0)
    X[4, 1] = np.float32(1e-42)  # denormal: bit-exact
    path = tmp_path / "d.mfad"
    V.save_dataset(path, X)
    raw = path.read_bytes()
    # io.cpp:91-104: "MFAD", u32 version 1, u64 N, u32 D, u8 dtype 0, 7 reserved, f32 rows (LE)
    want = b"MFAD" + struct.pack("<IQIB", 1, 37, 5, 0) + b"\0" * 7 + X.astype("<f4").tobytes()
    assert raw == want
    assert V.dataset_info(path) == (37, 5)
    Y = V.load_dataset(path)
    assert Y.tobytes() == X.tobytes()
    np.testing.assert_array_equal(V.load_dataset(path, 10, 7).view(np.uint32), X[10:17].view(np.uint32))


def test_mfam_layout_and_round_trip(tmp_path):
    p = _params(4, 6, 3)
    path = tmp_path / "m.mfam"
    V.save_checkpoint(path, p)
    raw = path.read_bytes()
    # io.cpp:127-149: "MFAM", u32 version, C, D, H, pi, mu, Lambda row-major D x H per component, dnoise
    lam_rowmajor = np.transpose(p.lam, (0, 2, 1))  # (C, D, H)
    want = (b"MFAM" + struct.pack("<IIII", 1, 4, 6, 3) + p.pi.astype("<f8").tobytes()
            + p.mu.astype("<f8").tobytes() + np.ascontiguousarray(lam_rowmajor).astype("<f8").tobytes()
            + p.psi.astype("<f8").tobytes())
    assert raw == want
    q = V.load_checkpoint(path)
    for f in ("pi", "mu", "lam", "psi"):
        assert getattr(q, f).tobytes() == getattr(p, f).tobytes(), f


def test_mfak_state_sidecar(tmp_path):
    rng = np.random.default_rng(2)
    K = np.sort(rng.choice(20, size=(50, 3), replace=True), axis=1).astype(np.int32)
    g = rng.integers(-1, 20, size=(20, 4)).astype(np.int32)
    gc = rng.integers(1, 5, size=20).astype(np.int32)
    path = tmp_path / "s.mfak"
    V.save_state(path, V.State(K, g, gc))
    st = V.load_state(path)
    assert np.array_equal(st.K, K) and np.array_equal(st.g, g) and np.array_equal(st.g_count, gc)
    sh = V.load_state(path, 20, 10)
    assert np.array_equal(sh.K, K[20:30]) and np.array_equal(sh.g, g)


def test_container_errors(tmp_path):
    X = np.ones((4, 3), np.float32)
    good = tmp_path / "d.mfad"
    V.save_dataset(good, X)
    raw = good.read_bytes()
    bad = tmp_path / "bad.mfad"
    bad.write_bytes(b"MFAX" + raw[4:])
    with pytest.raises(V.VmfaError, match="BadMagic"):
        V.load_dataset(bad)
    bad.write_bytes(raw[:-5])
    with pytest.raises(V.VmfaError, match="TruncatedFile"):
        V.load_dataset(bad)
    bad.write_bytes(raw[:2])
    with pytest.raises(V.VmfaError, match="TruncatedFile"):
        V.dataset_info(bad)
    bad.write_bytes(raw[:4] + struct.pack("<I", 2) + raw[8:])
    with pytest.raises(V.VmfaError, match="UnsupportedVersion"):
        V.load_dataset(bad)
    bad.write_bytes(raw[:20] + b"\x01" + raw[21:])  # dtype 1
    with pytest.raises(V.VmfaError, match="UnsupportedVersion"):
        V.load_dataset(bad)
    with pytest.raises(V.VmfaError, match="IoError"):
        V.load_dataset(tmp_path / "missing.mfad")
    with pytest.raises(V.VmfaError, match="InvalidArgument"):
        V.load_dataset(good, 2, 5)  # beyond the file's rows
    # MfaParams::validate before writing (model.cpp:14-41)
    p = _params(3, 4, 2)
    p.pi[0] += 1e-6
    with pytest.raises(V.VmfaError, match="InvalidArgument: mixing proportions do not sum to 1"):
        V.save_checkpoint(tmp_path / "m.mfam", p)
    p = _params(3, 4, 2)
    p.psi[1, 1] = 0.0
    with pytest.raises(V.VmfaError, match="noise variance"):
        V.save_checkpoint(tmp_path / "m.mfam", p)
    p = _params(3, 4, 2)
    V.save_checkpoint(tmp_path / "m.mfam", p)
    mraw = (tmp_path / "m.mfam").read_bytes()
    (tmp_path / "m2.mfam").write_bytes(mraw[:4] + struct.pack("<IIII", 1, 3, 4, 5) + mraw[20:])  # H > D
    with pytest.raises(V.VmfaError, match="IoError"):
        V.load_checkpoint(tmp_path / "m2.mfam")
