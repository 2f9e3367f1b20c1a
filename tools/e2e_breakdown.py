"""Wall-clock split of bench.py's e2e step (diagnostics): upload X / params /
state, iterate, download params / state, each timed on the host."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2501_12299_b200 import vmfa as V  # noqa: E402

X = V.gen_synthetic(V.synth_spec(2))
m = V.CONFIGS[2]["model"]
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
for it in range(2):
    s.variational_e_step(0, it)


def pin(a):
    b = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype))).pin_memory().numpy()
    b[...] = a
    return b


Xp = pin(X)
pp = V.Params(pin(p.pi), pin(p.mu), pin(p.lam), pin(p.psi))
sp = V.State(pin(st.K), pin(st.g), pin(st.g_count), pin(np.zeros(X.shape[0], np.int32)))
acc = {}
s.set_lookahead(os.environ.get("E2E_LOOKAHEAD", "0") == "1")
for i in range(8):
    marks = [("start", time.perf_counter())]
    s.upload_params(pp)
    marks.append(("upload_params", time.perf_counter()))
    s.upload_state(sp)
    marks.append(("upload_state", time.perf_counter()))
    s.upload_data(Xp, asynchronous=os.environ.get("E2E_ASYNC", "1") == "1")
    marks.append(("upload_data", time.perf_counter()))
    s.profile(i == 7)
    s.iterate(0, 100 + i)
    marks.append(("iterate", time.perf_counter()))
    s.download_params(out=pp)
    marks.append(("download_params", time.perf_counter()))
    s.download_state(out=sp)
    marks.append(("download_state", time.perf_counter()))
    if i >= 3:
        for (_, t0), (k, t1) in zip(marks, marks[1:]):
            acc[k] = acc.get(k, 0.0) + (t1 - t0) * 1e3 / 5
tot = sum(acc.values())
for k, v in acc.items():
    print(f"{k:16s} {v:7.3f} ms")
print(f"{'total':16s} {tot:7.3f} ms")
print({k: round(v["ms"], 3) for k, v in s.kernel_times().items()})
