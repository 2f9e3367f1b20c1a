"""Diagnostics: run config-2 iterations as bench.py does until an M-step fails,
then compare the failing component's statistics with the fp64 oracle's on the
same E-step output (tools only; not part of the product)."""
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2501_12299_b200 import vmfa as V  # noqa: E402
from paper_2501_12299_b200.abi import VmfaError  # noqa: E402

cfg = 2
m = V.CONFIGS[cfg]["model"]
X = V.gen_synthetic(V.synth_spec(cfg))
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1, loading_init=1)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
it = 0
for _ in range(2):
    s.variational_e_step(0, it)
    it += 1
fail = None
for step in range(int(os.environ.get("STEPS", "80"))):
    pc = s.download_params()
    kc = O.Caches(**s.download_caches())
    s.variational_e_step(0, it)
    it += 1
    s.accumulate_suffstats()
    try:
        s.update_params()
        s.truncated_free_energy()
    except VmfaError as ex:
        fail = ex
        print("step", step, "failed:", ex)
        break
if fail is None:
    print("no failure")
    sys.exit(0)
c = int(str(fail).split()[-1]) if str(fail).split()[-1].isdigit() else None
es = s.download_estep()
sn = s.download_state()
sd = s.download_suffstats()
resp = es[3]
so = O.accumulate_suffstats(X, pc, kc, sn.K, resp, threads=os.cpu_count())
H1 = m["H"] + 1
for name, a, b in (("Nc", sd.Nc[c], so.Nc[c]),):
    print(name, a, b)
Eg, Eo = sd.E[c], so.E[c]
print("E dev diag", np.diag(Eg))
print("E orc diag", np.diag(Eo))
print("max |dE|", np.abs(Eg - Eo).max(), "max |E|", np.abs(Eo).max())
print("eig dev", np.linalg.eigvalsh(Eg))
print("eig orc", np.linalg.eigvalsh(Eo))
rows = np.nonzero((sn.K == c).any(axis=1))[0]
q = resp[rows][sn.K[rows] == c]
print("rows with c in K:", rows.size, "resp: max", q.max() if q.size else None, "sum", q.sum())
print("psi range of c", pc.psi[c].min(), pc.psi[c].max(), "floor min", floor.min())
print("Sz eig", np.linalg.eigvalsh(kc.Sz[c]))
try:
    O.update_params(so, X.shape[0], pc, floor)
    print("oracle update on oracle stats: OK")
except Exception as ex:
    print("oracle update on oracle stats:", ex)
try:
    O.update_params(sd, X.shape[0], pc, floor)
    print("oracle update on device stats: OK")
except Exception as ex:
    print("oracle update on device stats:", ex)
