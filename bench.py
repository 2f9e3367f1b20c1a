"""bench.py — v-MFA EM iterations on B200 (BASELINE.json metric: candidate
log-joint evaluations/sec and EM iteration time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

A step is one main-loop iteration of train_vmfa (trainer.cpp:149-160): the
variational E-step (candidates, Woodbury log-joints, top-C', labels, g update,
responsibilities), sufficient statistics, update_params, precompute and the
post-M-step truncated free energy, over BASELINE config 2 (configs[1]: N=200k,
D=256, C=1000, H=8, C'=5, G=10) on synthetic data of that generator. value =
joint evaluations (sum_n |S(n)|, the reference counter) of all ranks per
second of the max-over-ranks device time. Under torchrun each rank holds its
own config-2-sized shard (weak scaling) and the ranks exchange the
co-occurrence table and the statistics with NCCL all-reduces.

--impl reference times the reference algorithm's CPU restatement (oracle/, the
reference library needs Eigen3, absent here) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate log-joint evals/sec & EM iteration time"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override rows per rank (testing only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-exact-ll", action="store_true")
    ap.add_argument("--profile-only", action="store_true",
                    help="run warm-up + 2 steps only (for ncu launch lists)")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]), src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, src="fallback")


class ClockSampler:
    """SM clocks and throttle reasons sampled by NVML every 5 ms during the
    timed region (nvidia-smi's loop mode is too coarse for a ~100 ms region);
    falls back to one nvidia-smi sample per boundary when NVML is missing."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.t = None

    def _sample_nvml(self, nv, h):
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for name, const in self.REASONS:
            if r & getattr(nv, const, 0):
                self.reasons.add(name)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return self._smi()
        while True:
            try:
                self._sample_nvml(nv, h)
            except Exception:
                break
            if self.stop.wait(self.period):
                break

    def _smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown," \
            "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
            "clocks_event_reasons.sw_power_cap"
        while True:
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                r = [x.strip() for x in out.split(",")]
                self.sm.append(float(r[0]))
                self.mx.append(float(r[1]))
                for (name, _), v in zip(self.REASONS, r[2:6]):
                    if v.lower() == "active":
                        self.reasons.add(name)
            except Exception:
                return
            if self.stop.wait(0.05):
                return

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=15)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def build_problem(cfg: int, rank: int, world: int, n_override: int = 0):
    from paper_2501_12299_b200 import vmfa as V
    m = V.CONFIGS[cfg]["model"]
    per = n_override or V.CONFIGS[cfg]["truth"]["N"]
    n_total = per * world
    spec = V.synth_spec(cfg, N=n_total)
    X = V.gen_synthetic(spec)
    p, st, floor, _ = V.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1,
                                   loading_init=1)
    a, b = rank * n_total // world, (rank + 1) * n_total // world
    return V, m, X, p, st, floor, a, b, n_total


def alg_per_joint(D, H):
    """F_j = 2DH + 3D + 2H flops, B_j = 4D + 8 bytes per joint."""
    return 2 * D * H + 3 * D + 2 * H, 4 * D + 8


def count_launches(sess, step_fn):
    """Kernels launched by one step, counted by the CUDA profiler (CUPTI via
    torch.profiler): every kernel in the process, ours and cub's."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step_fn()
        torch.cuda.synchronize()
    n = 0
    names = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" and not e.name.startswith("Memcpy") and not e.name.startswith("Memset"):
            n += 1
            names[e.name] = names.get(e.name, 0) + 1
    return n, names


def cpu_baseline_port(cfg: int, steps: int = 1, rows: int = 20000, threads: int = 0):
    """The reference algorithm restated (oracle/) on the host cores: full
    iterations on the first `rows` rows of the config's data with full C."""
    from oracle import oracle as O
    from paper_2501_12299_b200 import vmfa as V
    m = V.CONFIGS[cfg]["model"]
    threads = threads or os.cpu_count() or 1
    X = V.gen_synthetic(V.synth_spec(cfg), 0, rows)
    p, st, floor, _ = O.initialize(X, m["C"], m["H"], m["Cprime"], m["G"], seed=0, scale=0.1,
                                   loading_init=1)
    k = O.precompute_all(p)
    for it in range(2):  # warm-up E-steps, as in the GPU arm
        O.variational_e_step(X, p, k, st, 0, it, threads=threads)
    it = 2
    times, joints = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        e = O.variational_e_step(X, p, k, st, 0, it, threads=threads)
        s = O.accumulate_suffstats(X, p, k, st.K, e.resp, threads=threads)
        p = O.update_params(s, X.shape[0], p, floor)
        k = O.precompute_all(p)
        O.truncated_free_energy(X, p, k, st.K, threads=threads)
        times.append(time.perf_counter() - t0)
        joints.append(e.joints)
        it += 1
    return dict(value=float(sum(joints) / sum(times)), unit="joint evals/s", cores=threads,
                kind="port", iter_s=float(np.mean(times)),
                sample=f"config {cfg}, first {rows} rows, full C={m['C']}, {steps} full EM iteration(s) "
                       f"(E-step+stats+update+precompute+F) after 2 warm-up E-steps, {threads} threads")


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU restatement on the host
    cores (rank 0 only)."""
    if rank != 0:
        return
    from paper_2501_12299_b200 import vmfa as V
    m = V.CONFIGS[args.config]["model"]
    D, H = V.CONFIGS[args.config]["truth"]["D"], m["H"]
    rows = 20000
    cb = cpu_baseline_port(args.config, steps=max(1, args.steps), rows=rows)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "joint evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["iter_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config generator)",
        "config": {"workload": f"config{args.config} sample: {rows} rows, C={m['C']}, D={D}, H={H}, "
                               f"C'={m['Cprime']}, G={m['G']}"},
        "cpu_baseline": {"value": cb["value"], "unit": "joint evals/s", "cores": cb["cores"],
                         "kind": "port", "sample": cb["sample"]},
        "e2e": {"value": cb["value"], "unit": "joint evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "note": "reference library unbuildable (needs Eigen3, absent); timed = oracle/ fp64 "
                "restatement of the same algorithm, plain loops, std::thread with the reference chunking",
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2501_12299_b200 import vmfa as V
    V_, m, X, p, st, floor, a, b, n_total = build_problem(args.config, rank, world, args.n)
    D = X.shape[1]
    C, H, Cp, G = m["C"], m["H"], m["Cprime"], m["G"]
    sess = V.Session(C, D, H, Cp, G, X[a:b], n_offset=a, n_total=n_total, device=local)
    sess.set_floor(floor)
    sess.upload_params(p)
    sess.upload_state(V.State(st.K[a:b].copy(), st.g, st.g_count))
    ext = torch.cuda.ExternalStream(sess.stream())

    class _View:
        def __init__(self, ptr, n, dt):
            self.__cuda_array_interface__ = dict(shape=(n,), typestr="<i8" if dt == 0 else "<f8",
                                                 data=(ptr, False), version=3)

    xb = {}
    sparse = world > 1 and sess.cooc_sparse()
    if world > 1:
        for w in ((1, 2) if sparse else (0, 1, 2)):
            xb[w] = torch.as_tensor(_View(*sess.exchange_buffer(w)), device=f"cuda:{local}")

    def allreduce(w):
        with torch.cuda.stream(ext):
            if w == 0 and sparse:  # large C: owner-routed (c, c~) lists + int32 all-reduce of g
                from paper_2501_12299_b200.exchange import cooc_exchange
                cooc_exchange(sess, rank, world)
            else:
                dist.all_reduce(xb[w])
        ext.synchronize()

    it_counter = [0]

    def warm_estep():
        if world > 1:
            sess.phase_estep_local(0, it_counter[0])
            allreduce(0)
            sess.phase_estep_finish()
        else:
            sess.variational_e_step(0, it_counter[0])
        it_counter[0] += 1

    def step():
        it = it_counter[0]
        it_counter[0] += 1
        if world == 1:
            return sess.iterate(0, it)
        sess.phase_estep_local(0, it)
        allreduce(0)
        sess.phase_estep_finish()
        sess.phase_stats_local()
        allreduce(1)
        sess.phase_update()
        sess.phase_free_energy_local()
        allreduce(2)
        Fe, J, F = sess.phase_scalars()
        return dict(F_estep=Fe, joints=J, F=F)

    # the reference trainer's minimum warm-up: 2 E-steps
    for _ in range(2):
        warm_estep()
    for _ in range(args.warmup):
        step()
    if args.profile_only:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        return

    # L2 flush buffer (> 126 MB L2), written between timed iterations
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    times, joints, Fs = [], [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(ext):
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            r = step()
            e1.record(ext)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
            joints.append(r["joints"])
            Fs.append(r["F"])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # phase split: the same steps again with per-phase events (outside the timed region)
    sess.profile(True)
    for _ in range(args.steps):
        with torch.cuda.stream(ext):
            flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    kt = sess.kernel_times()
    sess.profile(False)
    ms_step = float(np.sum(times) / args.steps)
    J_rank = float(np.sum(joints) / args.steps)  # after the all-reduce J is already the job total
    if dist:
        t = torch.tensor([ms_step], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    J_job = J_rank if world > 1 else J_rank
    value = J_job / (ms_step * 1e-3)

    # dominant kernel: the candidate scoring (anchor + extra launches) of each E-step
    Fj, Bj = alg_per_joint(D, H)
    pk = peaks()
    sc_ms = (kt["score_anchor"]["ms"] + kt["score_extra"]["ms"]) / args.steps
    J_local = J_rank if world == 1 else J_rank / world
    ach_gbs = J_local * Bj / (sc_ms * 1e-3) / 1e9 if sc_ms > 0 else None
    ach_tfs = J_local * Fj / (sc_ms * 1e-3) / 1e12 if sc_ms > 0 else None
    phase_ms = {k: v["ms"] / args.steps for k, v in kt.items()}

    # exact log-likelihood (all N x C pairs, dense
    # tcgen05 pass) once after the timed region, on device time
    exact = None
    if not args.no_exact_ll:
        try:
            sess.exact_log_likelihood()  # first call allocates its buffers
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            ll = sess.exact_log_likelihood()
            e1.record(ext)
            e1.synchronize()
            t = e0.elapsed_time(e1)
            pairs = float(b - a) * C
            exact = {"ms": t, "log_likelihood": ll, "joints": pairs, "joints_per_s": pairs / (t * 1e-3),
                     "achieved_tflops": pairs * Fj / (t * 1e-3) / 1e12,
                     "roof_ms": max((b - a) * D * 4 / (pk["hbm"] * 1e9), pairs * Fj / (pk["bf16"] * 1e12 / 3)) * 1e3,
                     "roof": "max(X once at HBM peak, N*C*F_j at bf16-dense/3 (3-pass fp16 split))",
                     "how": "one vmfa_exact_log_likelihood call (images, row-tile-major dense jobs, "
                            "per-row LSE, fixed-order sum) between CUDA events"}
        except Exception as ex:
            exact = {"error": str(ex)}
    # SURVEY §8(f) item 1, second half: em_full_step (mstep.cpp:164-208) --
    # every pair's log-joint, full responsibilities and statistics
    em = None
    if not args.no_exact_ll:
        try:
            sess.em_full_step()  # first call allocates its buffers
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ext)
            ll, jn = sess.em_full_step()
            e1.record(ext)
            e1.synchronize()
            t = e0.elapsed_time(e1)
            em = {"ms": t, "log_likelihood": ll, "joints": jn, "joints_per_s": jn / (t * 1e-3),
                  "how": "one vmfa_em_full_step call (dense log-joints, q for all N x C pairs, statistics "
                         "over every pair) between CUDA events; not part of the timed v-MFA step"}
        except Exception as ex:
            em = {"error": str(ex)}

    # launches per step (CUPTI), outside the timed region
    n_launch, names = count_launches(sess, step)

    e2e = None
    if not args.no_e2e and world == 1:
        e2e = measure_e2e(V, sess, X[a:b], p, st, floor, args, ext)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline_port(args.config)
            cpu.pop("iter_s", None)
        except Exception as ex:  # the baseline is reported, never required
            cpu = {"error": str(ex)}

    # iteration-level roofline: T_roof = sum over phases of
    # max(F / P_pipe, B / BW) against the measured EM iteration time
    clk_sum = clk.summary()
    fp32_peak = 148 * 128 * 2 * (clk_sum.get("sm_max_mhz") or 1965.0) * 1e6  # FFMA, estimate (not in MEASURED_PEAKS)
    tc_peak = pk["bf16"] * 1e12 / 3  # 3-pass split fp16 MMA (fp16 dense = bf16 dense)
    bw = pk["hbm"] * 1e9
    n_loc = b - a
    Fm, Bm = 4 * D * H + 5 * D + 3 * H * H, 4 * D + 12
    roof = {
        "scoring": max(J_local * Fj / tc_peak, J_local * Bj / bw),
        "F_recompute": max(n_loc * Cp * Fj / tc_peak, n_loc * Cp * Bj / bw),
        "statistics": max(n_loc * Cp * Fm / fp32_peak, n_loc * Cp * Bm / bw),
        "update_precompute": C * (4 * D * H * H + 2 * D * (H + 1) ** 2 + H ** 3) / fp32_peak,
    }
    t_roof = sum(roof.values())
    # the statistics pass (the other large kernel) against its own roof
    st_ms = phase_ms.get("stats", 0.0)
    stats_roof = None
    if st_ms > 0:
        pairs = n_loc * Cp
        stats_roof = {"kernel": "statistics (k_stats + reduce + uncenter + Sigma_z)", "ms": st_ms,
                      "achieved_gbs": pairs * Bm / (st_ms * 1e-3) / 1e9, "peak_gbs": pk["hbm"],
                      "frac_hbm": pairs * Bm / (st_ms * 1e-3) / 1e9 / pk["hbm"],
                      "achieved_tflops": pairs * Fm / (st_ms * 1e-3) / 1e12,
                      "fp32_peak_tflops_est": fp32_peak / 1e12,
                      "frac_fp32": pairs * Fm / (st_ms * 1e-3) / fp32_peak,
                      "per_unit": f"B_m = 4D+12 = {Bm} B, F_m = 4DH+5D+3H^2 = {Fm} flop per (n, c in K(n)) pair "
                                  f"(SURVEY §8(d)), {pairs} pairs"}
    iter_roof = {"t_roof_ms": t_roof * 1e3, "t_iter_ms": ms_step, "frac": t_roof * 1e3 / ms_step,
                 "phases_ms": {k: v * 1e3 for k, v in roof.items()},
                 "how": "SURVEY §8(d): per phase max(F/P_pipe, B/BW); scoring/F at J and N*C' joints "
                        "(F_j, B_j), statistics at N*C' pairs (F_m = 4DH+5D+3H^2, B_m = 4D+12); "
                        "BW = measured HBM peak; P_pipe = bf16 dense / 3 for the split-fp16 scorer, "
                        "FFMA 148*128*2*f_max (estimate) elsewhere; F recompute is counted although "
                        "this build reads F from the next anchor pass"}

    traffic = {}
    try:
        with open(os.path.join(ROOT, "profiles", "scorer_traffic.json")) as f:
            traffic = json.load(f) if args.config == 2 else {}
    except Exception:
        pass
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "joint evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (BASELINE config generator, seeded), random-points init",
            "config": {"workload": f"config{args.config}: N={b - a} rows/GPU (N_total={n_total}), "
                                   f"D={D}, C={C}, H={H}, C'={Cp}, G={G}; one EM main iteration "
                                   f"per step (E-step, stats, update, precompute, truncated F)",
                       "l2": "flushed (256 MB write) before every timed iteration",
                       "parallelism": f"dp{world} (rows sharded, params replicated)"},
            "joints_per_step": J_job, "F_last": Fs[-1],
            "em_iteration_ms": ms_step,
            "phase_ms": phase_ms,
            "roofline": {"bound": "hbm", "kernel": "candidate scoring (score_anchor+score_extra)",
                         "achieved": ach_gbs, "peak": pk["hbm"], "unit": "GB/s",
                         "frac": (ach_gbs / pk["hbm"]) if ach_gbs else None,
                         "traffic": traffic.get("bytes_per_launch_pair"),
                         "traffic_src": traffic.get("source"), "peak_src": pk["src"],
                         "per_unit": f"B_j = 4D+8 = {Bj} B per joint (SURVEY §8(d)), J={J_local:.0f} joints per launch pair",
                         "flops_view": {"achieved_tflops": ach_tfs, "F_j": Fj}},
            "iteration_roofline": iter_roof,
            "roofline_statistics": stats_roof,
            "exact_ll": exact,
            "em_full_step": em,
            "gpu_launches": int(n_launch * args.steps),
            "launches_per_step": n_launch,
            "clocks": clk_sum,
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    sess.close()
    if dist:
        dist.destroy_process_group()


def measure_e2e(V, sess, Xs, p, st, floor, args, ext):
    """The same metric through the public API with host buffers: every step
    uploads the shard's rows, the parameters and the variational state from
    pinned host memory, runs the iteration and downloads the new parameters,
    state and labels into pinned host memory (the buffers the next step
    uploads from)."""
    import torch

    def pinned_like(a):
        return torch.empty(a.shape, dtype=getattr(torch, str(a.dtype))).pin_memory().numpy()

    def pin(a):
        b = pinned_like(np.ascontiguousarray(a))
        b[...] = a
        return b

    Xp = pin(Xs)
    pp = V.Params(pin(p.pi), pin(p.mu), pin(p.lam), pin(p.psi))
    sp = V.State(pin(st.K[:Xs.shape[0]]), pin(st.g), pin(st.g_count), pinned_like(np.zeros(Xs.shape[0], np.int32)))
    h2d = Xp.nbytes + sum(a.nbytes for a in (pp.pi, pp.mu, pp.lam, pp.psi, sp.K, sp.g, sp.g_count))
    d2h = sum(a.nbytes for a in (pp.pi, pp.mu, pp.lam, pp.psi, sp.K, sp.g, sp.g_count, sp.labels)) + 24
    ts, js = [], []
    it = 1000
    # the state is re-uploaded every step, so the next E-step's anchor pass
    # cannot be reused: F gets its own one-component pass (same value)
    sess.set_lookahead(False)
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sess.upload_params(pp)
        sess.upload_state(sp)
        sess.upload_data(Xp, asynchronous=True)  # overlaps the E-step's X-free prefix
        r = sess.iterate(0, it)
        sess.download_params(out=pp)
        sess.download_state(out=sp)
        t1 = time.perf_counter()
        it += 1
        if i >= args.warmup:
            ts.append(t1 - t0)
            js.append(r["joints"])
    sess.set_lookahead(True)
    return {"value": float(np.sum(js) / np.sum(ts)), "unit": "joint evals/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": float(np.mean(ts) * 1e3),
            "how": "host wall clock around upload(X, params, state) + iterate + download(params, state, labels, F), "
                   "pinned host buffers; X uploaded asynchronously (vmfa_upload_data_async), lookahead off"}


if __name__ == "__main__":
    main()
