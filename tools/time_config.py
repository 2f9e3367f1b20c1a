import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2501_12299_b200 import vmfa as V
cfg = 4
m = V.CONFIGS[cfg]["model"]
X = V.gen_synthetic(V.synth_spec(cfg))
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor); s.upload_params(p); s.upload_state(st)
for it in range(2): s.variational_e_step(0, it)
for it in range(2, 8):
    t0 = time.perf_counter(); r = s.iterate(0, it); t1 = time.perf_counter()
    print(it, round((t1 - t0) * 1e3, 2), r["F"], flush=True)
s.profile(True)
s.iterate(0, 8)
print({k: round(v["ms"], 2) for k, v in s.kernel_times().items()})
