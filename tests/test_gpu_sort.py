"""The hand-written stable radix sort of the K1 inversion (vmfa_sort.cu)
against numpy's stable argsort, over sizes around the tile and scan-tile
boundaries, 1-4 digit passes, skewed and uniform keys, repeated to catch
nondeterminism."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bits,dist", [(1, 4, "u"), (31, 8, "u"), (4096, 10, "u"), (4097, 10, "u"),
                                         (30000, 10, "u"), (30000, 10, "skew"), (65536 * 4 + 17, 13, "u"),
                                         (1_000_000, 16, "u"), (1_000_000, 12, "skew"), (3_000_001, 24, "u"),
                                         (200_000, 32, "u")])
def test_radix_sort_matches_stable_argsort(gpu, n, bits, dist):
    from paper_2501_12299_b200.abi import lib
    import ctypes as C
    rng = np.random.default_rng(n + bits)
    hi = (1 << bits) if bits < 32 else (1 << 32)
    if dist == "u":
        keys = rng.integers(0, hi, n, dtype=np.uint64).astype(np.uint32)
    else:  # a few hot keys
        keys = np.minimum(rng.geometric(0.05, n) - 1, hi - 1).astype(np.uint32)
    ko = np.empty(n, np.uint32)
    vo = np.empty(n, np.int32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    differ = lib().vmfa_diag_radix_sort(p(keys), n, bits, p(ko), p(vo), 5)
    assert differ == 0
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(vo, order.astype(np.int32))
    assert np.array_equal(ko, keys[order])
