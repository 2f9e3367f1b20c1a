"""Per-role cycle breakdown of the warp-specialised scorer on a BASELINE config
(argv[1], default 2; argv[2] rows, default the config's N) (diagnostics; uses
vmfa_diag_scorer_cycles)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2501_12299_b200 import vmfa as V  # noqa: E402
from paper_2501_12299_b200.abi import lib  # noqa: E402

CFG = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ROWS = int(sys.argv[2]) if len(sys.argv) > 2 else 0
X = V.gen_synthetic(V.synth_spec(CFG, N=ROWS) if ROWS else V.synth_spec(CFG))
m = V.CONFIGS[CFG]["model"]
p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0)
s = V.Session(m["C"], X.shape[1], m["H"], m["Cprime"], m["G"], X)
s.set_floor(floor)
s.upload_params(p)
s.upload_state(st)
for it in range(4):
    s.iterate(0, it)
names = ["P wait acc", "P job sync", "P wait stage", "P wait rows", "M wait acc", "M wait full", "M issue",
         "E wait", "E work", "P split", "P tmem st"]
lib().vmfa_diag_scorer_cycles(1, None, 0)
out = np.zeros(16, np.uint64)
s.profile(True)
s.variational_e_step(0, 10)
kt = s.kernel_times()
lib().vmfa_diag_scorer_cycles(1, out.ctypes.data_as(C.c_void_p), 16)
lib().vmfa_diag_scorer_cycles(0, None, 0)
print({k: round(v["ms"], 3) for k, v in kt.items() if v["ms"] > 0})
tot_p = out[0:4].sum()
print("cycles per CTA-role (summed over CTAs; producer counters summed over 8 warps):")
for i, nme in enumerate(names):
    tot_p = out[0:4].sum() + out[9:11].sum()
    share = out[i] / (tot_p if (i < 4 or i >= 9) else (out[4:7].sum() if i < 7 else out[7:9].sum()))
    print(f"  {nme:14s} {int(out[i]):>16d}  share-in-role {share:6.3f}")

# timeline of CTA 0 (anchor launch): per chunk (producer got stage, producer
# arrived full, MMA saw full, MMA issued), cycles relative to the first event
DBG = int(os.environ.get("WS_DBG", "0"))
lib().vmfa_diag_scorer_cycles(1 | (DBG << 1), None, 0)
big = np.zeros(16 + 8 * 512, np.uint64)
s.variational_e_step(0, 11)
lib().vmfa_diag_scorer_cycles(1 | (DBG << 1), big.ctypes.data_as(C.c_void_p), big.size)
kt2 = s.kernel_times()
print("WS_DBG", DBG, {k: round(v["ms"], 3) for k, v in kt2.items() if v["ms"] > 0})
lib().vmfa_diag_scorer_cycles(0, None, 0)
print("role counters of this E-step (anchor + extra launches):")
tp2 = float(big[0:4].sum() + big[9:11].sum())
for i, nme in enumerate(names):
    den = tp2 if (i < 4 or i >= 9) else float(big[4:7].sum() if i < 7 else big[7:9].sum())
    print(f"  {nme:14s} {int(big[i]):>16d}  share-in-role {big[i] / den:6.3f}")
tr = big[16:].reshape(-1, 8).astype(np.int64)
n = int((tr[:, 3] > 0).sum())
t0 = tr[0, 0] if tr[0, 0] > 0 else tr[0, 1]
print("chunk  got_stage  arrived  mma_sawA mma_sawB  mma_issued  ldr_start ldr_issued ldr_done  (period)")
for i in range(min(n, 48)):
    r = tr[i] - t0
    per = tr[i, 1] - tr[i - 1, 1] if i else 0
    print(f"{i:5d} {r[0]:10d} {r[1]:8d} {r[4]:8d} {r[2]:8d} {r[3]:10d} {r[5]:9d} {r[7]:9d} {r[6]:8d}  {per:6d}")
