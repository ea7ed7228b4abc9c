"""Closed-loop verification under the disturbance-feedback policy, on the device.

Drop-in for ``scanmpc.rollout`` (rollout.py:1-180): same names, arguments,
record type and error messages.  ``closed_loop`` / ``closed_loop_batched``
run ``k_rollout`` (csrc/models.cu) through ``gsls_rollout``: one CTA per
(rollout, instance) steps the device model under
u_k = v_k + sum_{j<k} Phi^u_{k,j} w_hat_j, injects E d_k, reconstructs
w_hat_k = E^+ (x_{k+1} - f(x_k, u_k)) and evaluates the constraint and tube
checks (rollout.py:47-93).  E is state-independent for every device model;
its range-restricted pseudo-inverse (rollout.py:41-44) is a one-time host
SVD at workspace creation.

``sample_disturbance`` reproduces the reference's seeded numpy streams bit
for bit and therefore stays a host function; ``adversarial_rows`` and
``superposition_check`` are host diagnostics over O(N) small products.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import Context, resolve, stream_ptr, to_dev, to_host
from .engine import DeviceModel
from .sls import SlsResponse, ragged_to_cells

F32, F64 = torch.float32, torch.float64
PINV_TRUNCATION = 1e-10  # rollout.py:17
WNORM_TOL = 1e-9         # rollout.py:18 (applied in k_rollout)


@dataclass
class RolloutRecord:
    """rollout.py:21-38."""
    x: np.ndarray
    u: np.ndarray
    w: np.ndarray
    stage_g: np.ndarray
    terminal_g: np.ndarray
    tube_margin: np.ndarray
    safe: bool
    tube_ok: bool
    disturbance_model_violated: bool
    max_w_norm: float

    @property
    def min_margin(self) -> float:
        vals = [-self.stage_g.max()] if self.stage_g.size else []
        if self.terminal_g.size:
            vals.append(-float(self.terminal_g.max()))
        return float(min(vals)) if vals else np.inf


def _range_restricted_pinv(E: np.ndarray) -> np.ndarray:
    """rollout.py:41-44 (workspace setup, not the hot path)."""
    U, s, Vt = np.linalg.svd(E)
    keep = s >= PINV_TRUNCATION
    s_inv = np.where(keep, 1.0 / np.where(keep, s, 1.0), 0.0)
    return Vt.T @ (s_inv[:, None] * U.T)


class DeviceRollouts:
    """Workspace for ``rollouts`` disturbance sequences on each of ``batch`` nominal plans."""

    def __init__(self, model, N: int, batch: int, rollouts: int):
        n, m, c, nf = model.nx, model.nu, model.nc, model.nf
        self.dims = (n, m, c, nf, N)
        self.B, self.R = int(batch), int(rollouts)
        self.ctx = Context(n, m, c, nf, N, self.B)
        self.dm = DeviceModel(model, N)
        E = np.asarray(model.disturbance(np.zeros(n)), float)
        self.E_host = E
        self.E = to_dev(E, F64)
        self.Epinv = to_dev(_range_restricted_pinv(E), F64)
        dev = self.E.device
        B, R = self.B, self.R
        z = lambda *s, dt=F64: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        self.out = {"x": z(B, R, N + 1, n), "u": z(B, R, N, m), "w": z(B, R, N, n), "stage_g": z(B, R, N, c),
                    "terminal_g": z(B, R, nf), "tube_margin": z(B, R, N), "max_w_norm": z(B, R),
                    "flags": z(B, R, 3, dt=torch.int32)}
        self._o = nat.RolloutOut(**{k: (v.data_ptr() if v.numel() else None) for k, v in self.out.items()})

    def run(self, x, u, phi_u, disturbances, h=None, tol_lin: float = 1e-2) -> dict:
        """x (B,N+1,n), u (B,N,m) float64; phi_u (B, N(N+1)/2, m, n) float32 cells or None;
        disturbances (B,R,N,n) float64; h (B,N,c) float64 or None.  All CUDA tensors."""
        n, m, c, nf, N = self.dims
        B, R = self.B, self.R
        _shape(x, (B, N + 1, n), "x")
        _shape(u, (B, N, m), "u")
        _shape(disturbances, (B, R, N, n), "disturbances")
        if phi_u is not None:
            _shape(phi_u, (B, N * (N + 1) // 2, m, n), "phi_u")
        if h is not None:
            _shape(h, (B, N, c), "h")
        a = nat.RolloutArgs()
        a.model_id, a.params, a.cons_offset = self.dm.model_id, self.dm.params.data_ptr(), self.dm.cons_offset
        a.x, a.u = x.data_ptr(), u.data_ptr()
        a.phi_u = phi_u.data_ptr() if phi_u is not None else None
        a.E, a.E_pinv = self.E.data_ptr(), self.Epinv.data_ptr()
        a.disturbances = disturbances.data_ptr()
        a.h = h.data_ptr() if h is not None and h.numel() else None
        a.tol_lin = float(tol_lin)
        a.rollouts = R
        nat.check(self.ctx.lib.gsls_rollout(self.ctx.handle, ctypes.byref(a), ctypes.byref(self._o), stream_ptr()),
                  "rollout")
        return self.out


def _shape(t, shape, name):
    if tuple(t.shape) != tuple(shape) or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CUDA tensor of shape {tuple(shape)}, got "
                         f"{tuple(t.shape)}")


def _workspace(model, N, B, R, executor=None) -> DeviceRollouts:
    dev = resolve(executor)
    cache = dev.__dict__.setdefault("_rollout_ws", {})
    key = (id(model), N, B, R)
    ws = cache.get(key)
    if ws is None or ws.dm.model is not model:
        ws = DeviceRollouts(model, N, B, R)
        cache[key] = ws
    return ws


def _phi_u_cells(response, N, nx, nu):
    cells = getattr(response, "_cells", None)  # DeviceSlsResponse: already device cells
    if cells is not None and cells[1].is_cuda:
        return cells[1].reshape(1, -1, nu, nx).contiguous()
    return to_dev(ragged_to_cells(response.Phi_u, N, (nu, nx)), F32)[None].contiguous()


def closed_loop_batched(model, x, u, phi_u, disturbances, h=None, tol_lin: float = 1e-2, executor=None) -> dict:
    """Batched rollout.closed_loop on device tensors (see DeviceRollouts.run); returns the
    workspace's output tensors: x, u, w, stage_g, terminal_g, tube_margin, max_w_norm, flags."""
    B, R, N = disturbances.shape[0], disturbances.shape[1], disturbances.shape[2]
    ws = _workspace(model, N, B, R, executor)
    return ws.run(x, u, phi_u, disturbances, h, tol_lin)


def closed_loop(model, traj, response, disturbances: np.ndarray, tightening=None, tol_lin: float = 1e-2,
                executor=None) -> RolloutRecord:
    """rollout.py:47-93 for one disturbance sequence."""
    N, nx, nu = traj.N, model.nx, model.nu
    disturbances = np.asarray(disturbances, float)
    if disturbances.shape != (N, nx):
        raise ValueError(f"disturbances must be ({N}, {nx})")
    ws = _workspace(model, N, 1, 1, executor)
    if not np.array_equal(np.asarray(model.disturbance(traj.x[0]), float), ws.E_host):
        raise TypeError(f"{type(model).__name__}: state-dependent disturbance maps have no device rollout")
    phiu = _phi_u_cells(response, N, nx, nu) if response is not None else None
    h = to_dev(np.asarray(tightening.h, float), F64)[None].contiguous() if tightening is not None else None
    o = ws.run(to_dev(np.asarray(traj.x, float), F64)[None].contiguous(),
               to_dev(np.asarray(traj.u, float), F64)[None].contiguous(), phiu,
               to_dev(disturbances, F64)[None, None].contiguous(), h, tol_lin)
    host = {k: to_host(v[0, 0]) for k, v in o.items()}
    fl = host["flags"]
    return RolloutRecord(x=host["x"], u=host["u"], w=host["w"], stage_g=host["stage_g"],
                         terminal_g=host["terminal_g"], tube_margin=host["tube_margin"], safe=bool(fl[0]),
                         tube_ok=bool(fl[1]), disturbance_model_violated=bool(fl[2]),
                         max_w_norm=float(host["max_w_norm"]))


def sample_disturbance(kind: str, n_x: int, horizon: int, seed, rows: np.ndarray | None = None) -> np.ndarray:
    """rollout.py:96-123; the seeded default_rng streams, identical to the reference."""
    rng = np.random.default_rng(seed)
    if kind == "uniform_ball":
        d = rng.standard_normal((horizon, n_x))
        d /= np.maximum(np.linalg.norm(d, axis=1, keepdims=True), 1e-300)
        return d * rng.random((horizon, 1)) ** (1.0 / n_x)
    if kind == "boundary":
        d = rng.standard_normal((horizon, n_x))
        return d / np.maximum(np.linalg.norm(d, axis=1, keepdims=True), 1e-300)
    if kind == "adversarial":
        if rows is None:
            raise ValueError("adversarial sampling needs per-stage constraint rows")
        rows = np.asarray(rows, float)
        if rows.shape != (horizon, n_x):
            raise ValueError(f"rows must be ({horizon}, {n_x})")
        norms = np.linalg.norm(rows, axis=1, keepdims=True)
        return np.divide(rows, norms, out=np.zeros_like(rows), where=norms > 1e-12)
    raise ValueError(f"unknown disturbance kind {kind!r}")


def adversarial_rows(model, traj, constraint_row: int | None = None, max_lookahead: int = 4) -> np.ndarray:
    """Per-stage push directions toward the nearest constraint boundary (rollout.py:126-166).

    Row k is the first nonzero (C_t A_{t-1} ... A_{k+1} E_k)^T over the look-ahead stages
    t = k+1 .. min(k + max_lookahead, N), where C_t is the state part of stage t's most
    violated constraint (or ``constraint_row``).  The model's Jacobians are evaluated once
    per stage along the trajectory (t = 1 .. N, with u_{N-1} at t = N) and every stage's
    window is one pass of running products over them.
    """
    N, nx = traj.N, model.nx
    x, u = np.asarray(traj.x, float), np.asarray(traj.u, float)
    ut = lambda t: u[min(t, N - 1)]  # noqa: E731
    push = [None] * (N + 1)  # push[t]: the selected state row of stage t's constraints, or None
    for t in range(1, N + 1):
        C, _ = model.stage_constraint_jacobians(x[t], ut(t))
        C = np.asarray(C, float)
        if not C.shape[0]:
            continue
        if constraint_row is not None:
            push[t] = C[constraint_row]
            continue
        live = np.flatnonzero(np.abs(C).sum(axis=1) > 1e-12)
        if live.size:
            g = np.asarray(model.stage_constraints(x[t], ut(t)), float)
            push[t] = C[live[np.argmax(g[live])]]
    A = [None] + [np.asarray(model.jacobians(x[t], ut(t))[0], float) for t in range(1, N)]
    rows = np.zeros((N, nx))
    for k in range(N):
        E = np.asarray(model.disturbance(x[k]), float)
        c_row = None  # C_t A_{t-1} ... A_{k+1}, built right to left
        for t in range(k + 1, min(k + max_lookahead, N) + 1):
            c_row = None if push[t] is None else push[t].copy()
            if c_row is not None:
                for s in range(t - 1, k, -1):
                    c_row = c_row @ A[s]
                cand = c_row @ E
                if np.linalg.norm(cand) > 1e-9:
                    rows[k] = cand
                    break
    return rows


def superposition_check(traj, response: SlsResponse, w: np.ndarray, realized_x: np.ndarray) -> float:
    """Worst |x_k - x_nom_k - sum_{j<k} Phi^x_{k,j} w_j| (rollout.py:169-180), all k at once:
    the response's lower-triangular blocks contracted with the disturbance sequence."""
    N = traj.N
    w = np.asarray(w, float)
    off = np.asarray(realized_x, float)[1:] - np.asarray(traj.x, float)[1:]
    pred = np.zeros_like(off)
    for j in range(N):  # column j feeds stages k = j+1 .. N
        pred[j:] += np.einsum("kab,b->ka", response.Phi_x[j], w[j])
    return float(np.abs(off - pred).max()) if N else 0.0
