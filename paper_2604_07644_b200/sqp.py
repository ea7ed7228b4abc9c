"""Drop-in for ``scanmpc.sqp``: Gauss-Newton SQP / RTI on the GPU.

Same dataclasses and entry points as /root/reference/pkg/src/scanmpc/sqp.py:
``Trajectory`` (:27-43), ``SqpSettings`` (:46-56), ``SqpStats`` (:59-67),
``NmpcResult`` / ``RtiResult`` (:70-86), ``initial_guess`` (:89-102),
``linearize`` (:105-147), ``solve_nmpc`` (:190-269), ``rti_step`` (:272-302).

Linearization, trajectory evaluation (defect / violation / l1 merit) and the
QP run on the device (csrc/models.cu, csrc/admm.cu); the host keeps the
SQP control flow (acceptance test, forcing of the inner tolerance, divergence
counter), reading back a handful of scalars per iteration.  Plants need a
device twin (``Model.device_spec``); there is no host evaluation path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native as nat
from . import admm as admm_mod
from .admm import AdmmSettings, AdmmState, DeviceAdmmState, DeviceAdmmStats, export_solution
from .device import Context, resolve, stream_ptr, to_dev, to_host
from .engine import DeviceModel, alloc_qp, linearize_into
from .errors import DivergenceError  # noqa: F401
from .lqr import LtvQpData
from .scan import scan_depth

F64 = torch.float64


@dataclass
class Trajectory:
    x: np.ndarray   # (N+1, nx)
    u: np.ndarray   # (N, nu)
    dt: float

    @property
    def N(self) -> int:
        return self.u.shape[0]

    def applied(self, dx, du, alpha: float) -> "Trajectory":
        return Trajectory(x=self.x + alpha * dx, u=self.u + alpha * du, dt=self.dt)

    def shifted(self) -> "Trajectory":
        x = np.vstack([self.x[1:], self.x[-1:]])
        u = np.vstack([self.u[1:], self.u[-1:]]) if self.N > 1 else self.u.copy()
        return Trajectory(x=x, u=u, dt=self.dt)


@dataclass
class SqpSettings:
    max_sqp_iters: int = 50
    kkt_tol: float = 1e-6
    line_search: bool = True
    alpha_min: float = 1e-3
    admm: AdmmSettings = field(default_factory=AdmmSettings)

    def __post_init__(self):
        if self.kkt_tol <= 0:
            raise ValueError("kkt_tol must be positive")


@dataclass
class SqpStats:
    iterations: int = 0
    converged: bool = False
    residual: float = np.inf
    admm_iterations: int = 0
    cost: float = np.nan
    scan_layers: int = 0
    admm_converged: bool = True
    # extension (not in the reference dataclass): one (iterations, converged, rho_changes,
    # cache_builds) record per inner admm.solve_qp call, for parity checks and profiling
    qp_calls: list = field(default_factory=list)


@dataclass
class NmpcResult:
    trajectory: Trajectory
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: SqpStats
    qp: LtvQpData | None = None


@dataclass
class RtiResult:
    u0: np.ndarray
    warm_start: Trajectory
    plan: Trajectory
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: SqpStats


def initial_guess(model, x0, N: int, mode: str = "hold") -> Trajectory:
    """sqp.py:89-102 (cold-start helper)."""
    x0 = np.asarray(x0, float)
    u = np.zeros((N, model.nu))
    if mode == "hold":
        x = np.tile(x0, (N + 1, 1))
    elif mode == "rollout":
        x = np.zeros((N + 1, model.nx))
        x[0] = x0
        for k in range(N):
            x[k + 1] = model.step(x[k], u[k])
    else:
        raise ValueError(f"unknown initial guess mode {mode!r}")
    return Trajectory(x=x, u=u, dt=model.dt)


class _Sqp:
    """Per (model, N) device workspace for batch-1 SQP / RTI calls."""

    def __init__(self, model, N: int):
        n, m, c, nf = model.nx, model.nu, model.nc, model.nf
        self.dims = (n, m, c, nf, N)
        self.ctx = Context(n, m, c, nf, N, 1)
        self.dm = DeviceModel(model, N)
        self.qp = alloc_qp(1, n, m, c, nf, N)
        self.E = torch.zeros(1, N, n, n, dtype=torch.float32, device=self.qp.QN.device)
        self.evals = torch.zeros(1, 8, dtype=F64, device=self.qp.QN.device)
        self.written = False

    def args(self, x, u, h=None, hf=None, xbar0=None):
        a = nat.LinArgs()
        a.model_id, a.params, a.cons_offset = self.dm.model_id, self.dm.params.data_ptr(), self.dm.cons_offset
        a.x, a.u = x.data_ptr(), u.data_ptr()
        a.h = h.data_ptr() if h is not None and h.numel() else None
        a.hf = hf.data_ptr() if hf is not None and hf.numel() else None
        a.xbar0 = xbar0.data_ptr() if xbar0 is not None else None
        a.Qw, a.Rw, a.QNw = self.dm.Qw.data_ptr(), self.dm.Rw.data_ptr(), self.dm.QNw.data_ptr()
        a.xref, a.uref, a.E_const = self.dm.xref.data_ptr(), self.dm.uref.data_ptr(), self.dm.E.data_ptr()
        a.write_weights = 1
        return a

    def linearize(self, traj, tight=None, xbar0=None):
        x, u = to_dev(traj.x, F64)[None], to_dev(traj.u, F64)[None]
        h, hf = _tight_dev(tight)
        xb = to_dev(xbar0, F64)[None] if xbar0 is not None else None
        linearize_into(self.ctx, self.dm, self.qp, x, u, h, hf, xb, self.E, write_weights=not self.written)
        self.written = True
        return x, u

    def export_qp(self, x_bar0=None) -> LtvQpData:
        """Host copy of the QP data held in the device buffers (last linearization)."""
        nat.check(self.ctx.lib.gsls_ctx_check(self.ctx.handle, stream_ptr()), "linearize")
        q = self.qp
        h = lambda t: to_host(t[0])  # noqa: E731
        return LtvQpData(A=h(q.A), B=h(q.B), b=h(q.b), Q=h(q.Q), R=h(q.R), S=h(q.S), q=h(q.q), r=h(q.r),
                         QN=h(q.QN), qN=h(q.qN), C=h(q.C), D=h(q.D), f=h(q.f), CN=h(q.CN), fN=h(q.fN),
                         dx0=h(q.dx0) if x_bar0 is not None else np.zeros(self.dims[0]))

    def evaluate(self, traj, tight=None, xbar0=None) -> np.ndarray:
        x, u = to_dev(traj.x, F64)[None], to_dev(traj.u, F64)[None]
        h, hf = _tight_dev(tight)
        xb = to_dev(xbar0, F64)[None] if xbar0 is not None else None
        a = self.args(x, u, h, hf, xb)
        nat.check(self.ctx.lib.gsls_traj_eval(self.ctx.handle, ctypes.byref(a), self.evals.data_ptr(),
                                              stream_ptr()), "traj_eval")
        return self.evals[0].cpu().numpy()

    def admm(self, settings: AdmmSettings, warm: AdmmState | None):
        n, m, c, nf, N = self.dims
        mtot = N * c + nf
        st = warm if warm is not None else AdmmState.fresh(mtot, settings.rho0)
        dst = DeviceAdmmState(1, mtot, st.rho)
        dst.load(0, st)
        dx, du, stats = admm_mod.solve_batched(self.ctx, self.qp, settings, dst, DeviceAdmmStats(1))
        dst.store(0, st)
        return dx, du, st, stats


def _tight_dev(tight):
    if tight is None:
        return None, None
    return to_dev(tight.h, F64)[None], to_dev(tight.hf, F64)[None]


def _workspace(model, N: int, executor=None) -> _Sqp:
    dev = resolve(executor)
    cache = dev.__dict__.setdefault("_sqp_ws", {})
    key = (id(model), N)
    ws = cache.get(key)
    if ws is None or ws.dm.model is not model:
        ws = _Sqp(model, N)
        cache[key] = ws
    return ws


def linearize(model, traj: Trajectory, tightenings=None, x_bar0=None, executor=None) -> LtvQpData:
    """Stagewise QP data around ``traj`` (sqp.py:105-147), evaluated on the device."""
    ws = _workspace(model, traj.N, executor)
    ws.linearize(traj, tightenings, x_bar0)
    return ws.export_qp(x_bar0)


def solve_nmpc(model, x_bar0, settings: SqpSettings, initial: Trajectory, tightenings=None, executor=None,
               warm_admm: AdmmState | None = None) -> NmpcResult:
    """Full SQP solve to the stated residual tolerance (sqp.py:190-269).

    Raises DivergenceError after five consecutive rejected steps; ADMM
    non-convergence is reported through stats.
    """
    x_bar0 = np.asarray(x_bar0, float)
    traj = initial
    ws = _workspace(model, traj.N, executor)
    n, m, c, nf, N = ws.dims
    stats = SqpStats()
    ast = warm_admm
    lam_s, lam_t = np.zeros((N, c)), np.zeros(nf)
    bad = 0
    scale = 1.0
    have_qp = False
    for _ in range(settings.max_sqp_iters):
        inner = settings.admm if scale == 1.0 else replace(
            settings.admm, tol_primal=settings.admm.tol_primal * scale, tol_dual=settings.admm.tol_dual * scale)
        ws.linearize(traj, tightenings, x_bar0)
        dx_t, du_t, ast, dstats = ws.admm(inner, ast)
        rec = torch.stack([dstats.iterations, dstats.converged, dstats.rho_changes, dstats.cache_builds]).cpu()
        its = int(rec[0, 0])
        stats.qp_calls.append(tuple(int(v) for v in rec[:, 0]))
        stats.admm_iterations += its
        stats.admm_converged = stats.admm_converged and bool(rec[1, 0])
        have_qp = True
        stats.scan_layers = scan_depth(N + 1)
        lam_s, lam_t = ast.lam[: N * c].reshape(N, c), ast.lam[N * c:]
        dx, du = to_host(dx_t[0]), to_host(du_t[0])
        ev = ws.evaluate(traj, tightenings, x_bar0)
        step = max(float(np.abs(dx).max(initial=0.0)), float(np.abs(du).max(initial=0.0)))
        resid = max(step, ev[1], max(ev[3], 0.0), ev[6])
        stats.residual = resid
        if resid <= settings.kkt_tol:
            stats.converged = True
            break
        alpha = 1.0
        if settings.line_search:
            K, k, P, p = export_solution(ws.ctx)
            cost = (P[0].double() @ dx_t[0][..., None])[..., 0] + p[0]
            mu = float(cost.abs().max()) if cost.numel() else 0.0
            weight = max(1.0, 10.0 * float(np.abs(ast.lam).max(initial=0.0)), 10.0 * mu)
            merit0 = ev[0] + weight * (ev[5] + ev[2] + ev[4])
            q, r, qN = to_host(ws.qp.q[0]), to_host(ws.qp.r[0]), to_host(ws.qp.qN[0])
            slope = float((q * dx[:-1]).sum() + (r * du).sum() + qN @ dx[-1])
            while True:
                e2 = ws.evaluate(traj.applied(dx, du, alpha), tightenings, x_bar0)
                if e2[0] + weight * (e2[5] + e2[2] + e2[4]) <= merit0 + 1e-4 * alpha * min(slope, 0.0):
                    break
                if alpha <= settings.alpha_min:
                    alpha = 0.0
                    break
                alpha *= 0.5
        stats.iterations += 1
        if alpha == 0.0:
            bad += 1
            if bad >= 5:
                raise DivergenceError("diverged")
            scale = max(scale * 0.1, 1e-4)
            continue
        bad = 0
        scale = 1.0
        traj = traj.applied(dx, du, alpha)
    stats.cost = float(ws.evaluate(traj)[0])
    # the last QP, as the reference returns it (sqp.py:268-269; None without an iteration)
    qp = ws.export_qp(x_bar0) if have_qp else None
    return NmpcResult(trajectory=traj, lam_stage=lam_s, lam_terminal=lam_t, stats=stats, qp=qp)


def rti_step(model, x_bar0, previous: Trajectory | None, settings: SqpSettings, tightenings=None, executor=None,
             warm_admm: AdmmState | None = None, horizon: int | None = None) -> RtiResult:
    """One linearize + QP + full step; returns u0 and the shifted warm start (sqp.py:272-302)."""
    x_bar0 = np.asarray(x_bar0, float)
    if previous is None:
        if horizon is None:
            raise ValueError("cold start needs a horizon")
        full = solve_nmpc(model, x_bar0, settings, initial_guess(model, x_bar0, horizon), tightenings, executor)
        plan = full.trajectory
        return RtiResult(u0=plan.u[0].copy(), warm_start=plan.shifted(), plan=plan, lam_stage=full.lam_stage,
                         lam_terminal=full.lam_terminal, stats=full.stats)
    ws = _workspace(model, previous.N, executor)
    n, m, c, nf, N = ws.dims
    ws.linearize(previous, tightenings, x_bar0)
    dx_t, du_t, ast, dstats = ws.admm(settings.admm, warm_admm)
    plan = previous.applied(to_host(dx_t[0]), to_host(du_t[0]), 1.0)
    conv = bool(dstats.converged[0])
    stats = SqpStats(iterations=1, converged=conv, residual=max(ast.r_primal, ast.r_dual),
                     admm_iterations=int(dstats.iterations[0]), scan_layers=scan_depth(N + 1),
                     admm_converged=conv, cost=float(ws.evaluate(plan)[0]))
    return RtiResult(u0=plan.u[0].copy(), warm_start=plan.shifted(), plan=plan,
                     lam_stage=ast.lam[: N * c].reshape(N, c), lam_terminal=ast.lam[N * c:], stats=stats)
