"""Max relative errors of the device statistics (Y, E, sq, N_c) against the
fp64 oracle on a few shapes, for the selected kernel (VMFA_STATS=ffma: k_stats,
default: k_stats_mma). Diagnostics only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from _helpers import gaussian_problem, to_vmfa_params, to_vmfa_state  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

for (N, D, C, H, Cp, G) in [(20000, 256, 20, 8, 5, 10), (4000, 64, 40, 4, 3, 5), (5000, 40, 30, 3, 3, 5),
                            (3000, 256, 30, 15, 3, 5), (3000, 784, 24, 16, 5, 10), (3000, 64, 30, 16, 3, 5)]:
    X, _ = gaussian_problem(N, D, max(4, C // 2), min(H, 4), seed=5)
    p, st, floor, _ = O.initialize(X, C, H, Cp, G, seed=0, scale=0.1, loading_init=1)
    s = V.Session(C, D, H, Cp, G, X)
    s.set_floor(floor)
    s.upload_params(to_vmfa_params(V, p))
    s.upload_state(to_vmfa_state(V, st))
    s.variational_e_step(0, 0)
    _, _, _, resp = s.download_estep()
    stg = s.download_state()
    so = O.accumulate_suffstats(X, p, O.precompute_all(p), stg.K, resp, threads=8)
    s.accumulate_suffstats()
    sg = s.download_suffstats()

    def rel(a, b, atol=0.0):
        # error / the test's tolerance (rtol 1e-5 + atol): <= 1 passes test_mstep_parity
        return float((np.abs(a - b) / (1e-5 * np.abs(b) + atol + 1e-300)).max())
    print(f"N={N} D={D} C={C} H={H} (error / tolerance): Nc {rel(sg.Nc, so.Nc) / 10:.3f}"
          f"  E {rel(sg.E, so.E, 1e-6 * np.abs(so.E).max()):.3f}"
          f"  Y {rel(sg.Y, so.Y, 1e-6 * np.abs(so.Y).max()):.3f}  sq {rel(sg.sq, so.sq):.3f}", flush=True)
    s.close()
