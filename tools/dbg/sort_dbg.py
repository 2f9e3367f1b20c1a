import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2501_12299_b200.abi import lib
p = lambda a: a.ctypes.data_as(C.c_void_p)
for n, bits in [(4097, 10), (8192, 8), (8192, 9), (4097, 8), (12288, 4)]:
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 1 << bits, n).astype(np.uint32)
    order = np.argsort(keys, kind="stable")
    for rep in range(4):
        ko = np.empty(n, np.uint32); vo = np.empty(n, np.int32)
        lib().vmfa_diag_radix_sort(p(keys), n, bits, p(ko), p(vo), 1)
        bad = np.nonzero(vo != order)[0]
        print(n, bits, rep, "bad", len(bad), bad[:8], vo[bad[:4]], order[bad[:4]], "keys ok", np.array_equal(np.sort(ko), np.sort(keys)))
