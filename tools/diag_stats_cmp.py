"""Config-2 statistics: the tensor-core kernel vs the FFMA kernel on the same
device state, iteration by iteration (diagnostics)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m = V.CONFIGS[cfg]["model"]
X = V.gen_synthetic(V.synth_spec(cfg))
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
for it in range(2):
    s.variational_e_step(0, it)
for it in range(2, 8):
    out = {}
    for k in ("ffma", "mma"):
        if k == "ffma":
            os.environ["VMFA_STATS"] = "ffma"
        else:
            os.environ.pop("VMFA_STATS", None)
        s.accumulate_suffstats()
        out[k] = s.download_suffstats()
    a, b = out["mma"], out["ffma"]
    for f in ("Nc", "E", "Y", "sq"):
        x, y = getattr(a, f), getattr(b, f)
        bad = ~np.isfinite(x)
        d = np.abs(x - y) / (1e-5 * np.abs(y) + 1e-6 * np.abs(y).max())
        w = np.unravel_index(np.argmax(np.where(np.isfinite(d), d, np.inf)), d.shape)
        print(it, f, "nonfinite", int(bad.sum()), "max err/tol", float(np.nanmax(d)), "at", w, flush=True)
    try:
        s.iterate(0, it)
    except Exception as e:
        print("iterate", it, "raised", e)
        break
