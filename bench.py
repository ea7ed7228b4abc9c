#!/usr/bin/env python
"""Benchmark: robust MPC steps (QP + SLS) on B200, BASELINE.json's metric.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--batch B]

Our arm (default): BASELINE cfg-D — one robust RTI step (sls.rti_robust_step:
linearize, SLS synthesis + tube tightening, tightened ADMM QP, duals) per
scenario for a batch of 1024 perturbed 61D-quadruped scenarios per GPU
(weak scaling; ranks all-gather one result record per instance with NCCL
after every step).  ``value`` is
whole-job solves/s timed with CUDA events; ``e2e`` is the same through the
public API with inputs copied from pinned host memory and u0/plan read
back every step.  Single-instance step latency p50/p90 at 61D and 75D is
reported alongside.  ``cpu_baseline`` times the CPU oracle (a float64
restatement of the reference, ``oracle/``) on the box's host cores.

Reference arm (--impl reference): the CPU oracle port of the reference
algorithm on the same workload, all host cores (one single-threaded solve
per core), rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MPC step latency ms p50 (QP+SLS) at 61D/75D; batched solves/sec at 1-8 GPUs"
UNIT = "solves/s"


# --------------------------------------------------------------------------- helpers

def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _admm_max_iter():
    from paper_2604_07644_b200 import scenarios
    return scenarios.ADMM["max_iter"]


def makespan_block(its_all, fam_s, iters_per_step, B, b_iter, hbm_peak, max_iter):
    """ADMM load balance: the per-instance iteration spread of the timed
    batch against the replay's device time, and the replay time the same total iteration
    count would take at the bulk waves' measured bandwidth (ncu, profiles/rNN/traffic.json)
    -- the excess is the long-running instances' tail (latency-bound clusters)."""
    it = its_all.flatten().cpu().numpy()
    q = np.percentile(it, [50, 90, 99])
    out = {"mean": float(it.mean()), "p50": float(q[0]), "p90": float(q[1]), "p99": float(q[2]),
           "max": float(it.max()), "at_max_iter_fraction": float((it >= max_iter).mean()),
           "iterations_in_instances_beyond_p90": float(it[it > q[1]].sum() / max(it.sum(), 1.0))}
    rep = fam_s.get("replay")
    tr = ncu_traffic().get("replay") or {}
    if rep and tr.get("duration_ms") and tr.get("units"):
        bulk_gbs = tr["units"] * b_iter / (tr["duration_ms"] / 1e3) / 1e9  # algorithmic, first (full) wave
        at_bulk_ms = iters_per_step * b_iter / (bulk_gbs * 1e9) * 1e3
        out.update({"replay_ms_per_step": rep[0], "bulk_wave_gbs": bulk_gbs,
                    "replay_ms_at_bulk_bandwidth": at_bulk_ms, "tail_excess_ms": rep[0] - at_bulk_ms})
    return out


def ncu_traffic():
    """DRAM bytes per launch of the roofline kernels from the committed ncu capture."""
    try:
        for rnd in ("r02", "r01"):  # the latest round's captures
            f = os.path.join(ROOT, "profiles", rnd, "traffic.json")
            if os.path.exists(f):
                return json.load(open(f))
    except Exception:
        pass
    return {}


def W(L):
    return 2 * (L - 1)


def flops_cvf(n):
    return 50.0 / 3.0 * n ** 3          # 16 2/3 n^3 per CVF combine (matrix part)


def flops_build(n, m, N):
    """SURVEY §8d F_build: one LQR cache build (CVF tree + COT tree + per-stage gains)."""
    return (W(N + 1) * (50.0 / 3.0 * n ** 3 + 8 * n * n) + W(N) * (2 * n ** 3 + 2 * n * n)
            + N * (14 * n * n * m + 8 * n * m * m + 2 * m ** 3))


def flops_sls(n, m, c, nf, N):
    """SURVEY §8d F_SLS: one SLS synthesis + tightening (N(N-1) CVF combines at 18 2/3 n^3 with
    the gains / closed loop, per-cell costs and row norms)."""
    V = N * (N - 1) / 2
    return (N * (N - 1) * 56.0 / 3.0 * n ** 3
            + V * (2 * m ** 3 + 16 * n * n * m + 10 * n * m * m + 2 * m * n * n + 2 * c * (2 * n * n + m * m + 2 * n * m))
            + 4 * N * nf * n * n)


def bytes_replay_iter(n, m, c, nf, N):
    """SURVEY §8d B_iter: algorithmic bytes of one cached ADMM iteration (fp32 convention)."""
    return 4 * (4 * n * n * W(N + 1) + n * n * W(N) + N * (n * n + 2 * m * m + 3 * n * m + 2 * c * (n + m) + 5 * n
                                                          + 3 * m + 5 * c) + 2 * nf * n)


# --------------------------------------------------------------------------- CPU arms

def _oracle_worker(args):
    """One oracle rti_robust_step of scenario `idx` (float64 numpy, one core); returns its
    wall time and the outputs the parity block compares with the GPU's instance `idx`."""
    tag, idx = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    from paper_2604_07644_b200 import scenarios
    import oracle
    wl = scenarios.rti_workload(tag)
    m = wl.model
    rs = oracle_settings(m)
    tau = oracle.sls.Duals.zero(wl.N, m.nc, m.nf, rs.eps)
    tau.tau = wl.tau
    tau.tau_term = wl.tau_term
    x = wl.scenario_states(idx, 1)[0]
    st = oracle.admm.State.fresh(wl.N * m.nc + m.nf, rs.sqp.admm.rho0)
    prev = oracle.sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    t = time.perf_counter()
    r = oracle.sls.rti_robust_step(m, x, prev, tau, rs, warm_admm=st)
    dt = time.perf_counter() - t
    qp = oracle.sqp.linearize(m, prev, r.tightening, x)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    return {"t": dt, "iters": r.stats.admm_iterations, "rho_changes": st.generation, "idx": idx,
            "active": st.z >= f - 1e-12, "u0": r.u0, "h": r.tightening.h, "hf": r.tightening.hf}


def parity_block(eng, res, first=0):
    """bench.py parity: the GPU instances `first + r['idx']` of the timed batch vs the oracle
    results `res` (same scenarios): ADMM iterations, rho changes and the active set exactly,
    u0 / h within 1e-4 (reference.relative_error)."""
    import oracle
    z = eng.state.z.cpu().numpy()
    f = np.concatenate([eng.qp.f.cpu().numpy().reshape(eng.B, -1), eng.qp.fN.cpu().numpy()], axis=1)
    its, rc = eng.stats.iterations.cpu().numpy(), eng.stats.rho_changes.cpu().numpy()
    u0, h = eng.u0.cpu().numpy(), eng.h.cpu().numpy()
    n_it = n_act = 0
    e_u0 = e_h = 0.0
    for r in res:
        i = r["idx"] - first
        n_it += int(its[i] == r["iters"] and rc[i] == r["rho_changes"])
        n_act += int(((z[i] >= f[i] - 1e-12) == r["active"]).all())
        e_u0 = max(e_u0, oracle.relative_error(u0[i], r["u0"]))
        e_h = max(e_h, oracle.relative_error(h[i], r["h"]))
    n = len(res)
    return {"instances": n, "checker": "oracle (float64 restatement of the reference, pinned by tests/golden)",
            "admm_iterations_and_rho_changes_exact": f"{n_it}/{n}", "active_set_exact": f"{n_act}/{n}",
            "u0_max_rel_err": e_u0, "h_max_rel_err": e_h, "tol": 1e-4,
            "pass": bool(n_it == n and n_act == n and e_u0 <= 1e-4 and e_h <= 1e-4)}


def oracle_settings(model):
    import oracle
    from paper_2604_07644_b200 import scenarios as S
    return oracle.sls.RobustSettings(
        sqp=oracle.sqp.Settings(admm=oracle.admm.Settings(**S.ADMM), **S.SQP), eps=S.EPS,
        weights=oracle.sls.Weights(np.eye(model.nx), S.RBAR * np.eye(model.nu), np.eye(model.nx)))


def cpu_round(pool, tag, first, count):
    t = time.perf_counter()
    res = pool.map(_oracle_worker, [(tag, first + i) for i in range(count)])
    return time.perf_counter() - t, res


def _worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"


def make_pool(cores):
    import multiprocessing as mp
    os.environ["OPENBLAS_NUM_THREADS"] = "1"   # inherited by the spawned workers before numpy loads
    ctx = mp.get_context("spawn")
    pool = ctx.Pool(cores, initializer=_worker_init)
    os.environ.pop("OPENBLAS_NUM_THREADS", None)
    return pool


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    pool = make_pool(cores)
    try:
        for w in range(args.warmup):
            cpu_round(pool, "q61", w * cores, cores)
        t_tot, n_tot = 0.0, 0
        per = []
        for k in range(args.steps):
            dt, res = cpu_round(pool, "q61", (args.warmup + k) * cores, cores)
            t_tot += dt
            n_tot += len(res)
            per.extend(r["t"] for r in res)
    finally:
        pool.close()
    value = n_tot / t_tot
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_tot / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args.batch, world),
           "latency_ms_p50": {"q61": 1e3 * statistics.median(per)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": f"{args.steps} rounds x {cores} q61 scenarios, one oracle rti_robust_step each "
                                      "(single-threaded numpy per core, multiprocessing pool)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------- GPU arm

def workload_config(batch, world):
    return {"workload": "cfg-D: 61D/12u synthetic quadruped, one robust RTI step (linearize + SLS synthesis/"
                        "tightening + tightened ADMM QP + duals) per scenario, N=25, nc=26, nf=2",
            "batch_per_gpu": batch, "N": 25, "nx": 61, "nu": 12, "parallelism": f"dp{world} (independent scenarios; "
            "one NCCL all_gather of a per-instance result record (u0, ADMM stats, cost) per step)", "l2": "inputs larger than L2 (per-step SLS/LQR workspace >> 126 MB)",
            "timing": "CUDA events on the launching stream, max over ranks"}


def latency(tag, steps=30, warmup=5):
    """Single-instance robust RTI step latency (device events) and through the drop-in API."""
    import torch
    from paper_2604_07644_b200 import scenarios, sls, sqp
    from paper_2604_07644_b200.engine import RtiEngine
    from paper_2604_07644_b200.sls import ragged_to_cells
    wl = scenarios.rti_workload(tag)
    m = wl.model
    rs = scenarios.our_settings()(m)
    eng = RtiEngine(m, wl.N, 1, rs)
    d = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    xb, px, pu = d(wl.xbar0[None]), d(wl.prev_x[None]), d(wl.prev_u[None])
    tc, tt = d(ragged_to_cells(wl.tau, wl.N, (m.nc,))[None]), d(wl.tau_term[None])
    times = []
    for i in range(warmup + steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        eng.step(xb, px, pu, tau=tc, tau_term=tt)
        e1.record()
        torch.cuda.synchronize()
        if i >= warmup:
            times.append(e0.elapsed_time(e1))
    its = int(eng.stats.iterations[0])
    # the same step recorded as one CUDA graph (RtiEngine.capture): one launch, no host sync;
    # its duals carry over from step to step (the engine-held tau), as in closed loop
    graph = {}
    try:
        cap = eng.capture(xb, px, pu)
        g_times = []
        for i in range(warmup + steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            cap()
            e1.record()
            torch.cuda.synchronize()
            if i >= warmup:
                g_times.append(e0.elapsed_time(e1))
        cap.check()
        graph = {"p50": statistics.median(g_times), "p90": float(np.percentile(g_times, 90)),
                 "admm_iterations": int(eng.stats.iterations[0]), "graph_launches_per_step": 1}
    except Exception as exc:  # noqa: BLE001 - reported, not hidden
        graph = {"error": f"{type(exc).__name__}: {exc}"}
    # per-kernel-family breakdown of the same step (separate, profiled pass)
    from paper_2604_07644_b200 import _native as nat
    lib = nat.load()
    lib.gsls_prof_enable(1)
    lib.gsls_prof_read(None, None, None, 0)
    for _ in range(5):
        eng.step(xb, px, pu, tau=tc, tau_term=tt)
    torch.cuda.synchronize()
    lib.gsls_prof_enable(0)
    nfam = len(nat.PROF_FAMILIES)
    pm, pl = np.zeros(nfam), np.zeros(nfam, np.int64)
    lib.gsls_prof_read(pm.ctypes.data, None, pl.ctypes.data, nfam)
    phases = {k: round(float(v) / 5, 4) for k, v, c in zip(nat.PROF_FAMILIES, pm, pl) if c}
    # end to end through the public drop-in API (numpy in, numpy out)
    tau = sls.SlsDuals.zero(wl.N, m.nc, m.nf, rs.eps)
    tau.tau, tau.tau_term = wl.tau, wl.tau_term
    prev = sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    e2e = []
    for i in range(warmup + steps // 2):
        t = time.perf_counter()
        sls.rti_robust_step(m, wl.xbar0, prev, tau, rs).u0
        torch.cuda.synchronize()
        if i >= warmup:
            e2e.append(1e3 * (time.perf_counter() - t))
    del eng
    return {"p50": statistics.median(times), "p90": float(np.percentile(times, 90)), "admm_iterations": its,
            "e2e_p50": statistics.median(e2e), "phases_ms": phases, "graph": graph}


PHASE_GROUPS = {"sls": ("sls_assemble", "sls_leaf", "sls_cvf", "sls_gains", "sls_matprod", "sls_phiu", "sls_rownorm",
                         "sls_small"),
                "build": ("leaf", "cvf_lqr", "gains", "cot"),
                "replay": ("replay",),
                "other": ("linearize", "rti_misc")}


def serialized_phases(eng, step, nat, lib, steps=2):
    """Per-family device time of the batched step with both overlaps off (the SLS / first-build
    side stream and the ADMM driver's rebuild side stream), so the families add up to the
    serialized step; returns (families, serialized ms per step, builds per step)."""
    import torch
    ov = eng.overlap
    eng.overlap = False
    os.environ["GSLS_ADMM_SERIAL"] = "1"
    try:
        step()
        torch.cuda.synchronize()
        lib.gsls_prof_enable(1)
        lib.gsls_prof_read(None, None, None, 0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        builds = 0
        e0.record()
        for _ in range(steps):
            step()
            builds += int(eng.stats.cache_builds.sum())
        e1.record()
        torch.cuda.synchronize()
        lib.gsls_prof_enable(0)
    finally:
        eng.overlap = ov
        os.environ.pop("GSLS_ADMM_SERIAL", None)
    nfam = len(nat.PROF_FAMILIES)
    pm, pu_, pl = np.zeros(nfam), np.zeros(nfam), np.zeros(nfam, np.int64)
    lib.gsls_prof_read(pm.ctypes.data, pu_.ctypes.data, pl.ctypes.data, nfam)
    fam = {k: (float(t) / steps, int(c) // steps) for k, t, c in zip(nat.PROF_FAMILIES, pm, pl) if c}
    return fam, e0.elapsed_time(e1) / steps, builds / steps


def phase_rooflines(fam, B, dims, iters_per_step, builds_per_step, fp32_peak, hbm_peak):
    """SURVEY §8d per-phase rooflines on the serialized family times: SLS and LQR-build flop
    against the FP32-SIMT peak, the cached ADMM iterations' bytes against HBM, and the
    time-weighted whole-step fraction (the 'other' phases count with fraction 0)."""
    n, m, c, nf, N = dims
    out, tw, tt = {}, 0.0, 0.0
    for ph, fams in PHASE_GROUPS.items():
        t = sum(fam[f][0] for f in fams if f in fam)
        if t <= 0:
            continue
        if ph == "sls":
            work, unit, peak, bound = flops_sls(n, m, c, nf, N) * B / 1e12, "TFLOP/s", fp32_peak, "fp32-simt"
        elif ph == "build":
            work, unit, peak, bound = flops_build(n, m, N) * builds_per_step / 1e12, "TFLOP/s", fp32_peak, "fp32-simt"
        elif ph == "replay":
            work, unit, peak, bound = bytes_replay_iter(n, m, c, nf, N) * iters_per_step / 1e9, "GB/s", hbm_peak, "hbm"
        else:
            work, unit, peak, bound = None, None, None, "latency"
        ach = work / (t / 1e3) if work is not None else None
        frac = ach / peak if ach is not None else 0.0
        out[ph] = {"ms_per_step": t, "bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": frac,
                   "families": {f: {"ms": fam[f][0], "launches": fam[f][1]} for f in fams if f in fam}}
        tw += t * frac
        tt += t
    out["time_weighted_frac"] = tw / tt if tt else None
    return out


def receding_horizon(tag, steps=200, warmup=10, seed=0, graph=False):
    """Closed-loop MPC at batch 1: each robust RTI step's u0 drives the plant (model.step plus a
    bounded disturbance E w, |w| <= 1), the next step warm-starts from the shifted plan and the
    engine-held duals.  Device time per step (CUDA events around RtiEngine.step) and the loop's
    wall time per step (incl. the u0 read-back and the host plant step)."""
    import torch
    from paper_2604_07644_b200 import scenarios
    from paper_2604_07644_b200.engine import RtiEngine
    from paper_2604_07644_b200.sls import ragged_to_cells
    wl = scenarios.rti_workload(tag)
    m = wl.model
    eng = RtiEngine(m, wl.N, 1, scenarios.our_settings()(m))
    d = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    rng = np.random.default_rng(seed)
    x = np.array(wl.xbar0, float)
    px, pu = d(wl.prev_x[None]), d(wl.prev_u[None])
    tc, tt = d(ragged_to_cells(wl.tau, wl.N, (m.nc,))[None]), d(wl.tau_term[None])
    dev_ms, wall_ms, its = [], [], []
    done = 0
    cap = None
    try:
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            xb = d(x[None])
            if graph and k == 1:  # record after the first (tau-seeding) eager step
                cap = eng.capture(xb, px, pu)
            e0.record()
            if k == 0:
                eng.step(xb, px, pu, tau=tc, tau_term=tt)
            elif cap is not None:
                cap(xb, px, pu)
            else:
                eng.step(xb, px, pu)
            e1.record()
            if cap is not None:
                cap.check()
            u0 = eng.u0[0].cpu().numpy()
            w = rng.standard_normal(m.nx)
            w *= rng.random() ** (1.0 / m.nx) / np.linalg.norm(w)
            x = np.asarray(m.step(x, u0), float) + np.asarray(m.disturbance(x), float) @ w
            px, pu = eng.warm_x.clone(), eng.warm_u.clone()
            if k >= warmup:
                dev_ms.append(e0.elapsed_time(e1))
                wall_ms.append(1e3 * (time.perf_counter() - t0))
                its.append(int(eng.stats.iterations[0]))
            done = k + 1
            if not np.all(np.isfinite(x)):
                break
    except Exception as exc:  # noqa: BLE001 - reported, not hidden
        return {"error": f"{type(exc).__name__}: {exc}", "steps_done": done}
    if not dev_ms:
        return {"error": "no timed steps", "steps_done": done}
    return {"steps": len(dev_ms), "device_ms_p50": statistics.median(dev_ms),
            "device_ms_p90": float(np.percentile(dev_ms, 90)), "device_ms_max": max(dev_ms),
            "loop_wall_ms_p50": statistics.median(wall_ms), "admm_iterations_mean": float(np.mean(its)),
            "admm_iterations_max": int(max(its)), "mode": "CUDA graph replay (one launch per step)" if graph else "eager",
            "disturbance": "x+ = f(x, u0) + E(x) w, w uniform in the unit ball (seed 0)"}


def cpu_latency(tag, steps=5, warmup=1):
    """Single-process CPU latency of one robust RTI step: the oracle (float64 numpy, the
    reference's algorithm) with numpy's BLAS threads on all host cores."""
    import oracle
    from paper_2604_07644_b200 import scenarios
    wl = scenarios.rti_workload(tag)
    m = wl.model
    rs = oracle_settings(m)
    tau = oracle.sls.Duals.zero(wl.N, m.nc, m.nf, rs.eps)
    tau.tau, tau.tau_term = wl.tau, wl.tau_term
    prev = oracle.sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    times = []
    for k in range(warmup + steps):
        t = time.perf_counter()
        oracle.sls.rti_robust_step(m, wl.xbar0, prev, tau, rs)
        if k >= warmup:
            times.append(1e3 * (time.perf_counter() - t))
    return {"p50_ms": statistics.median(times), "p90_ms": float(np.percentile(times, 90)), "steps": steps,
            "cores": os.cpu_count(), "kind": "port",
            "threads": "one process; numpy BLAS on all host cores (the reference's own executor threads engage only "
                       "at >= 64 combines per layer, scan.py:118-120)"}


def config_lines(reps=2):
    """BASELINE configs B, C, E through the drop-in API (host numpy in and out), wall ms."""
    import torch
    from paper_2604_07644_b200 import admm, scenarios as S, sls, sqp
    out = {}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            ts.append(1e3 * (time.perf_counter() - t))
        return r, min(ts)
    try:
        m = S.cfgb_model()
        x0 = S.quad12_start()
        xg, ug = S.hover_guess(m, x0, S.CFGB["N"])
        st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGB["admm"]), **S.CFGB["sqp"])
        r, ms = timed(lambda: sqp.solve_nmpc(m, x0, st, sqp.Trajectory(xg, ug, m.dt)))
        out["cfgB_solve_nmpc"] = {"ms": ms, "N": S.CFGB["N"], "nx": m.nx, "nu": m.nu, "sqp_iterations": r.stats.iterations,
                                  "admm_iterations": r.stats.admm_iterations, "converged": bool(r.stats.converged)}
        mc = S.cfgc_model()
        xg, ug = S.hover_guess(mc, x0, S.CFGC["N"])
        stc = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGC["admm"]), **S.CFGC["sqp"])
        rs = sls.RobustSettings(sqp=stc, weights=sls.SlsWeights.identity(mc.nx, mc.nu), eps=S.CFGC["eps"],
                                tol_h=S.CFGC["tol_h"], max_alternations=S.CFGC["max_alternations"])
        r, ms = timed(lambda: sls.solve_robust(mc, x0, rs, initial=sqp.Trajectory(xg, ug, mc.dt)))
        out["cfgC_solve_robust"] = {"ms": ms, "N": S.CFGC["N"], "alternations": r.stats.alternations,
                                    "sqp_iterations": r.stats.sqp_iterations, "converged": bool(r.stats.converged)}
        me = S.cfge_model()
        N = S.CFGE["N"]
        x, u = S.cfge_trajectory(me, N)
        qp = sqp.linearize(me, sqp.Trajectory(x, u, me.dt), None, S.cfge_start(me))
        ste = admm.AdmmSettings(**S.CFGE["admm"])
        r, ms = timed(lambda: admm.solve_qp(qp, ste))
        out["cfgE_solve_qp"] = {"ms": ms, "N": N, "nx": me.nx, "nu": me.nu,
                                "variables": (N + 1) * me.nx + N * me.nu, "constraints": N * qp.nc + qp.nf,
                                "admm_iterations": r.stats.iterations, "cache_builds": r.stats.cache_builds,
                                "converged": bool(r.stats.converged)}
    except Exception as exc:  # noqa: BLE001 - reported, not hidden
        out["error"] = f"{type(exc).__name__}: {exc}"
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2604_07644_b200 import _native as nat, scenarios
    from paper_2604_07644_b200.engine import RtiEngine
    from paper_2604_07644_b200.sls import ragged_to_cells

    rank, local, world = dist_env()
    # GSLS_BENCH_BACKEND=gloo (tests only): several ranks on one GPU, to check the multi-rank
    # control flow (barriers, max-over-ranks timing, rank-0-only passes) on a one-GPU box
    backend = os.environ.get("GSLS_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    lib = nat.load()
    peaks = measured_peaks()

    lat = {}
    if rank == 0 and not args.no_latency:
        for tag in ("q61", "h75"):
            lat[tag] = latency(tag)

    wl = scenarios.rti_workload("q61")
    m = wl.model
    B = args.batch
    n, mu, c, nf, N = m.nx, m.nu, m.nc, m.nf, wl.N
    rs = scenarios.our_settings()(m)
    eng = RtiEngine(m, N, B, rs)
    d = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    xs = wl.scenario_states(rank * B, B)   # weak scaling: rank r owns scenarios [rB, (r+1)B)
    host = {"xbar0": xs, "prev_x": np.broadcast_to(wl.prev_x, (B,) + wl.prev_x.shape).copy(),
            "prev_u": np.broadcast_to(wl.prev_u, (B,) + wl.prev_u.shape).copy(),
            "tau": np.broadcast_to(ragged_to_cells(wl.tau, N, (c,)), (B, N * (N + 1) // 2, c)).copy(),
            "tau_term": np.broadcast_to(wl.tau_term, (B, N, nf)).copy()}
    dev = {k: d(v) for k, v in host.items()}
    from paper_2604_07644_b200 import dist as D
    rec = torch.empty(B, mu + len(D.RESULT_FIELDS), dtype=torch.float64, device="cuda")
    gathered = torch.empty(world * B, rec.shape[1], dtype=torch.float64, device="cuda")

    def step(inp):
        eng.step(inp["xbar0"], inp["prev_x"], inp["prev_u"], tau=inp["tau"], tau_term=inp["tau_term"])
        if world > 1:   # the only collective: one record per instance (u0 + ADMM stats + cost)
            D.gather_results(D.pack_engine(eng, rec), world, out=gathered)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step(dev)
    torch.cuda.synchronize()
    barrier()

    # ---- timed: device-resident inputs ------------------------------------------
    lib.gsls_prof_enable(1)
    lib.gsls_prof_read(None, None, None, 0)
    its = []
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step(dev)
            its.append(eng.stats.iterations.clone())
        e1.record()
        torch.cuda.synchronize()
        barrier()
    lib.gsls_prof_enable(0)
    ms = e0.elapsed_time(e1)
    nfam = len(nat.PROF_FAMILIES)
    pm, pu_, pl = np.zeros(nfam), np.zeros(nfam), np.zeros(nfam, np.int64)
    lib.gsls_prof_read(pm.ctypes.data, pu_.ctypes.data, pl.ctypes.data, nfam)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t)
    value = world * B * args.steps / (ms_max / 1e3)
    its_all = torch.stack(its).double()

    # ---- timed: end to end through the API with host buffers ---------------------
    pinned = {k: torch.as_tensor(v).pin_memory() for k, v in host.items()}
    out_u0 = torch.empty(B, mu, dtype=torch.float64).pin_memory()
    out_plan = torch.empty(B, N + 1, n, dtype=torch.float64).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in pinned.values())
    d2h = out_u0.numel() * 8 + out_plan.numel() * 8
    def e2e_step():
        inp = {k: t.to("cuda", non_blocking=True) for k, t in pinned.items()}
        step(inp)
        out_u0.copy_(eng.u0, non_blocking=True)
        out_plan.copy_(eng.plan_x, non_blocking=True)
        torch.cuda.current_stream().synchronize()

    e2e_step()  # warm-up of the host-buffer path (its device input buffers come from the caching allocator)
    torch.cuda.synchronize()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record()
    for _ in range(args.steps):
        e2e_step()
    e3.record()
    torch.cuda.synchronize()
    barrier()
    ms_e = torch.tensor([e2.elapsed_time(e3)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_e, op=dist.ReduceOp.MAX)
    e2e_value = world * B * args.steps / (float(ms_e) / 1e3)

    # ---- closed-loop verification of the step's policies (rollout.py:47-93):
    #      S disturbance sequences per instance under the synthesized Phi^u, device-timed ------
    from paper_2604_07644_b200 import rollout as RO
    S_ro, K_ro = 16, 5
    _, phiu_cells, _ = eng.export_response()
    gen = torch.Generator(device="cuda").manual_seed(rank)
    dro = torch.randn(B, S_ro, N, n, dtype=torch.float64, device="cuda", generator=gen)
    dro /= dro.norm(dim=-1, keepdim=True)
    dro *= torch.rand(B, S_ro, N, 1, dtype=torch.float64, device="cuda", generator=gen) ** (1.0 / n)
    ro_ws = RO.DeviceRollouts(m, N, B, S_ro)
    ro_out = ro_ws.run(eng.plan_x, eng.plan_u, phiu_cells, dro, eng.h)
    torch.cuda.synchronize()
    e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e4.record()
    for _ in range(K_ro):
        ro_out = ro_ws.run(eng.plan_x, eng.plan_u, phiu_cells, dro, eng.h)
    e5.record()
    torch.cuda.synchronize()
    ro_ms = e4.elapsed_time(e5) / K_ro
    fl = ro_out["flags"].cpu().numpy()
    rollout_line = {"metric": "closed-loop rollouts/s (rollout.closed_loop under the step's Phi^u, h)",
                    "value": B * S_ro / (ro_ms / 1e3), "unit": "rollouts/s", "rollouts_per_call": B * S_ro,
                    "per_instance": S_ro, "N": N, "ms_per_call": ro_ms, "safe_fraction": float(fl[..., 0].mean()),
                    "tube_ok_fraction": float(fl[..., 1].mean()), "disturbances": "uniform unit ball, torch seed = rank",
                    "kernel": "k_rollout", "launches_per_call": 1}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- per-phase rooflines on a serialized pass (families add up to the step) ----------
    clk = clocks.summary()
    sm_max = clk["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    # FP32-SIMT peak: measured on a B200 of this pool (tools/micro/fp32peak.cu, committed result);
    # MEASURED_PEAKS.json carries no FP32-SIMT figure.  Fallback: 148 SMs x 128 FMA/clk x 2 x clock.
    fp32_src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "fp32_peak.json")
    try:
        with open(fp32_src) as fh:
            fp32_peak, fp32_how = float(json.load(fh)["fp32_ffma_tflops"]), "measured: profiles/r01/fp32_peak.json (tools/micro/fp32peak.cu)"
    except (OSError, ValueError, KeyError):
        fp32_peak, fp32_how = 148 * 128 * 2 * sm_max * 1e6 / 1e12, "derived: 148 SMs x 128 FP32 FMA/clk x 2 x max SM clock"
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    total_iters = float(its_all.sum())
    iters_per_step = total_iters / args.steps
    fam = dict(zip(nat.PROF_FAMILIES, zip(pm, pu_, pl)))  # timed loop: (ms, units, launches)
    fam_s, ms_serial, builds_per_step = serialized_phases(  # rank 0 alone from here: the step without its all-gather
        eng, lambda: eng.step(dev["xbar0"], dev["prev_x"], dev["prev_u"], tau=dev["tau"],
                              tau_term=dev["tau_term"]), nat, lib)
    dims = (n, mu, c, nf, N)
    rl_phase = phase_rooflines(fam_s, B, dims, iters_per_step, builds_per_step, fp32_peak, hbm_peak)
    tr = ncu_traffic()
    rl = {}
    for k in ("sls_cvf", "cvf_lqr"):
        if k in fam_s:
            t_ms, nl = fam_s[k]
            units = fam[k][1] / args.steps  # combines per step (the timed loop's unit count)
            ach = units * flops_cvf(n) / (t_ms / 1e3) / 1e12
            rl[k] = {"bound": "fp32-simt", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                     "ms_per_step": t_ms, "traffic": (tr.get(k) or {}).get("dram_bytes"),
                     "traffic_launch": (tr.get(k) or {}).get("launch")}
    if "replay" in fam_s:
        t_ms, nl = fam_s["replay"]
        ach = iters_per_step * bytes_replay_iter(n, mu, c, nf, N) / (t_ms / 1e3) / 1e9
        rl["replay"] = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                        "ms_per_step": t_ms, "traffic": (tr.get("replay") or {}).get("dram_bytes"),
                        "traffic_launch": (tr.get("replay") or {}).get("launch")}
    dom = max(fam_s, key=lambda k: fam_s[k][0])
    roof = dict(rl.get(dom, {}), kernel=dom,
                peak_source=fp32_how if dom in ("sls_cvf", "cvf_lqr") else "MEASURED_PEAKS.json hbm_gbs",
                work=("units = combines per launch x batch; 16 2/3 n^3 flop per combine (SURVEY §8d)"
                      if dom in ("sls_cvf", "cvf_lqr") else "B_iter x ADMM iterations (SURVEY §8d)"),
                timing="serialized pass (side streams off), CUDA events per kernel family")
    phases = {"serialized_ms_per_step": ms_serial, "families_sum_ms": sum(v[0] for v in fam_s.values()),
              "overlapped_ms_per_step": ms_max / args.steps,
              "families": {k: {"ms_per_step": v[0], "launches_per_step": v[1]} for k, v in fam_s.items()},
              "lqr_builds_per_step": builds_per_step}

    # ---- closed-loop latency, configs B / C / E ----------------------------------------
    rh = {}
    if not args.no_latency:
        for tag in ("q61", "h75"):
            rh[tag] = receding_horizon(tag, steps=args.rh_steps)
            rh[tag + "_graph"] = receding_horizon(tag, steps=args.rh_steps, graph=True)
    cfg_lines = config_lines() if not args.no_latency else {}

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------------
    cpu = None
    parity = None
    if world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        pool = make_pool(cores)
        try:
            dt, res = cpu_round(pool, "q61", 0, cores)
        finally:
            pool.close()
        cpu = {"value": len(res) / dt, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{cores} q61 scenarios, one oracle rti_robust_step each (single-threaded numpy per core)"}
        parity = parity_block(eng, res)
        cpu["latency_q61"] = cpu_latency("q61")

    launches = int(pl.sum())
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32 factorizations / f64 vectors", "data": "synthetic",
           "config": workload_config(B, world),
           "latency_ms_p50": {k: v["p50"] for k, v in lat.items()},
           "latency_ms_p90": {k: v["p90"] for k, v in lat.items()},
           "latency_e2e_ms_p50": {k: v["e2e_p50"] for k, v in lat.items()},
           "latency_admm_iterations": {k: v["admm_iterations"] for k, v in lat.items()},
           "latency_graph_ms": {k: v["graph"] for k, v in lat.items()},
           "latency_phases_ms": {k: v["phases_ms"] for k, v in lat.items()},
           "admm_iterations_mean": total_iters / its_all.numel(),
           "admm_makespan": makespan_block(its_all, fam_s, iters_per_step, B, bytes_replay_iter(n, mu, c, nf, N),
                                           hbm_peak, max_iter=_admm_max_iter()),
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
           "gpu_launches": launches, "roofline": roof, "roofline_by_kernel": rl, "roofline_by_phase": rl_phase,
           "phases": phases, "receding_horizon_b1": rh, "configs_drop_in": cfg_lines,
           "rollout": rollout_line,
           "clocks": {"sm_mhz": clk["sm_mhz"], "sm_max_mhz": clk["sm_max_mhz"], "reasons": clk["reasons"]},
           "cpu_baseline": cpu, "parity": parity}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--rh-steps", type=int, default=200)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
