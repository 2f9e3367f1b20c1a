"""Device time of E-steps (and of one full iteration, when it succeeds) for a
BASELINE config on a row subset: `python tools/time_estep.py CONFIG ROWS`.
Reports joints per E-step, ms, joints/s and the scoring roofline terms."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2501_12299_b200 import vmfa as V  # noqa: E402

cfg, rows = int(sys.argv[1]), int(sys.argv[2])
m = V.CONFIGS[cfg]["model"]
t0 = time.time()
X = V.gen_synthetic(V.synth_spec(cfg), 0, rows)
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
print("setup s", round(time.time() - t0, 1), flush=True)
out = {"config": cfg, "rows": rows, "C": m["C"], "D": X.shape[1], "H": m["H"], "estep": []}
ext = torch.cuda.ExternalStream(s.stream())
for it in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    F, J = s.variational_e_step(0, it)
    e1.record(ext)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    out["estep"].append({"ms": ms, "joints": int(J), "joints_per_s": J / (ms * 1e-3), "F": F})
    print(out["estep"][-1], flush=True)
s.profile(True)
s.variational_e_step(0, 4)
out["estep_phase_ms"] = {k: round(v["ms"], 3) for k, v in s.kernel_times().items() if v["ms"] > 0}
s.profile(False)
try:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    r = s.iterate(0, 5)
    e1.record(ext)
    e1.synchronize()
    out["iteration"] = {"ms": e0.elapsed_time(e1), "joints": r["joints"]}
    s.profile(True)
    s.iterate(0, 6)
    out["iteration_phase_ms"] = {k: round(v["ms"], 3) for k, v in s.kernel_times().items() if v["ms"] > 0}
    s.profile(False)
except Exception as ex:  # noqa: BLE001
    out["iteration"] = {"error": str(ex)}
print(json.dumps(out), flush=True)
