"""Drop-in for ``scanmpc.admm``: the inequality-constrained LTV-QP by ADMM on the GPU.

Same dataclasses and entry point as /root/reference/pkg/src/scanmpc/admm.py:
``AdmmSettings`` (:24-39), ``AdmmState`` (:42-55), ``AdmmStats`` (:58-67),
``AdmmResult`` (:70-79), ``solve_qp`` (:153-203), plus the stacking helpers
(:82-97) and the scalar ``update_rho`` rule (:138-150).

The whole iteration loop runs on the device (csrc/admm.cu): one persistent
CTA per instance replays the cached factorization every iteration, projects,
ascends the duals, reduces the residuals and applies the penalty rule; a
committed rho change returns control to the host driver, which rebuilds the
factorization for exactly those instances (admm.py:171-178) and resumes.
``warm_start`` is mutated in place and returned, as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import lqr
from .device import DeviceQp, resolve, stream_ptr, to_host
from .scan import scan_depth

RHO_GATE = 5.0


@dataclass
class AdmmSettings:
    rho0: float = 0.1
    rho_min: float = 1e-6
    rho_max: float = 1e6
    sigma: int = 10
    tol_primal: float = 1e-6
    tol_dual: float = 1e-6
    max_iter: int = 4000

    def __post_init__(self):
        if self.sigma < 2:
            raise ValueError("sigma must be >= 2")
        for name in ("rho0", "rho_min", "rho_max", "tol_primal", "tol_dual"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    def cstruct(self) -> nat.AdmmSettings:
        return nat.AdmmSettings(float(self.rho0), float(self.rho_min), float(self.rho_max), int(self.sigma),
                                float(self.tol_primal), float(self.tol_dual), int(self.max_iter))


@dataclass
class AdmmState:
    z: np.ndarray
    lam: np.ndarray
    y: np.ndarray
    rho: float
    generation: int = 0
    iteration: int = 0
    r_primal: float = np.inf
    r_dual: float = np.inf

    @classmethod
    def fresh(cls, m: int, rho: float) -> "AdmmState":
        return cls(z=np.zeros(m), lam=np.zeros(m), y=np.zeros(m), rho=rho)


@dataclass
class AdmmStats:
    iterations: int = 0
    converged: bool = False
    r_primal: float = np.inf
    r_dual: float = np.inf
    rho: float = 0.0
    rho_changes: int = 0
    cache_builds: int = 0
    scan_layers: int = 0


@dataclass
class AdmmResult:
    dx: np.ndarray
    du: np.ndarray
    state: AdmmState
    stats: AdmmStats
    solution: lqr.LqrSolution

    def stage_duals(self, qp):
        return split_stacked(qp, self.state.lam)


def stacked_offsets(qp) -> np.ndarray:
    """admm.py:82-83."""
    return np.concatenate([np.asarray(qp.f).ravel(), np.asarray(qp.fN)])


def split_stacked(qp, v):
    """admm.py:86-88."""
    nc, N = qp.nc, qp.N
    return v[: N * nc].reshape(N, nc), v[N * nc:]


def constraint_values(qp, dx, du) -> np.ndarray:
    """admm.py:91-97 (host helper for inspecting results)."""
    C, D, CN = (np.asarray(getattr(qp, k)) for k in ("C", "D", "CN"))
    dx, du = np.asarray(dx), np.asarray(du)
    if qp.N == 0:
        return CN @ dx[0] if qp.nf else np.zeros(0)
    stage = (C @ dx[:-1, :, None])[..., 0] + (D @ du[..., None])[..., 0]
    term = CN @ dx[-1] if qp.nf else np.zeros(0)
    return np.concatenate([stage.ravel(), term])


def update_rho(state: AdmmState, r_primal: float, r_dual: float, settings: AdmmSettings) -> AdmmState:
    """Residual balancing with the factor-5 gate (admm.py:138-150); the device applies the same rule."""
    ratio = np.sqrt(max(r_primal, 1e-30) / max(r_dual, 1e-30))
    proposed = float(np.clip(state.rho * ratio, settings.rho_min, settings.rho_max))
    if proposed > RHO_GATE * state.rho or proposed < state.rho / RHO_GATE:
        state.rho = proposed
        state.generation += 1
        state.y = state.lam / state.rho
    return state


class DeviceAdmmState:
    """Batched ADMM state in device memory (the gsls_admm_state_t buffers)."""

    def __init__(self, batch: int, m: int, rho0: float, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.z = torch.zeros(batch, m, dtype=torch.float64, device=dev)
        self.lam = torch.zeros_like(self.z)
        self.y = torch.zeros_like(self.z)
        self.rho = torch.full((batch,), float(rho0), dtype=torch.float64, device=dev)
        self.r_primal = torch.full((batch,), np.inf, dtype=torch.float64, device=dev)
        self.r_dual = torch.full_like(self.r_primal, np.inf)
        self.generation = torch.zeros(batch, dtype=torch.int32, device=dev)
        self.iteration = torch.zeros_like(self.generation)

    def cstruct(self) -> nat.AdmmState:
        s = nat.AdmmState()
        for k in ("z", "lam", "y", "rho", "r_primal", "r_dual", "generation", "iteration"):
            t = getattr(self, k)
            setattr(s, k, t.data_ptr() if t.numel() else None)
        return s

    def load(self, i: int, st: AdmmState):
        for k in ("z", "lam", "y"):
            getattr(self, k)[i] = torch.as_tensor(np.asarray(getattr(st, k), float), dtype=torch.float64)
        self.rho[i] = float(st.rho)
        self.generation[i] = int(st.generation)
        self.iteration[i] = int(st.iteration)
        self.r_primal[i] = float(st.r_primal)
        self.r_dual[i] = float(st.r_dual)

    def store(self, i: int, st: AdmmState):
        st.z, st.lam, st.y = (to_host(getattr(self, k)[i]) for k in ("z", "lam", "y"))
        st.rho = float(self.rho[i])
        st.generation = int(self.generation[i])
        st.iteration = int(self.iteration[i])
        st.r_primal = float(self.r_primal[i])
        st.r_dual = float(self.r_dual[i])


class DeviceAdmmStats:
    def __init__(self, batch: int, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        z = lambda: torch.zeros(batch, dtype=torch.int32, device=dev)  # noqa: E731
        self.iterations, self.converged, self.rho_changes, self.cache_builds = z(), z(), z(), z()

    def cstruct(self) -> nat.AdmmStats:
        return nat.AdmmStats(self.iterations.data_ptr(), self.converged.data_ptr(), self.rho_changes.data_ptr(),
                             self.cache_builds.data_ptr())


def solve_batched(ctx, dqp: DeviceQp, settings: AdmmSettings, state: DeviceAdmmState,
                  stats: DeviceAdmmStats | None = None):
    """Batched device ADMM on an existing context; returns (dx, du, stats) as tensors."""
    d = ctx.dims
    dev = dqp.QN.device
    stats = stats or DeviceAdmmStats(d.batch, dev)
    dx = torch.empty(d.batch, d.N + 1, d.nx, dtype=torch.float64, device=dev)
    du = torch.empty(d.batch, d.N, d.nu, dtype=torch.float64, device=dev)
    s, st, sa, ss = dqp.cstruct(), settings.cstruct(), state.cstruct(), stats.cstruct()
    rc = ctx.lib.gsls_admm_solve_qp(ctx.handle, ctypes.byref(s), ctypes.byref(st), ctypes.byref(sa),
                                    ctypes.byref(ss), dx.data_ptr(), du.data_ptr() if du.numel() else None,
                                    stream_ptr())
    nat.check(rc, "admm.solve_qp")
    return dx, du, stats


def export_solution(ctx):
    """K, k, P, p of the last solve held by ``ctx`` (tensors with a batch dim)."""
    d = ctx.dims
    dev = torch.device("cuda", torch.cuda.current_device())
    e = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
    e64 = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
    K, k, P, p = e(d.batch, d.N, d.nu, d.nx), e64(d.batch, d.N, d.nu), e(d.batch, d.N + 1, d.nx, d.nx), \
        e64(d.batch, d.N + 1, d.nx)
    rc = ctx.lib.gsls_ctx_export_solution(ctx.handle, K.data_ptr() if K.numel() else None,
                                          k.data_ptr() if k.numel() else None, P.data_ptr(), p.data_ptr(),
                                          stream_ptr())
    nat.check(rc, "export_solution")
    return K, k, P, p


def solve_qp(qp, settings: AdmmSettings | None = None, warm_start: AdmmState | None = None,
             executor=None) -> AdmmResult:
    """ADMM loop around the scan-LQR primal update (admm.py:153-203).

    Terminates when ||G - z||_inf <= tol_primal and rho ||z+ - z||_inf <= tol_dual;
    otherwise returns the last iterate with converged=False.
    """
    settings = settings or AdmmSettings()
    dev = resolve(executor)
    n, m, c, nf, N = qp.nx, qp.nu, qp.nc, qp.nf, qp.N
    mtot = N * c + nf
    ctx = dev.context(n, m, c, nf, N, 1)
    dqp = DeviceQp.from_host(qp)
    state = warm_start if warm_start is not None else AdmmState.fresh(mtot, settings.rho0)
    dstate = DeviceAdmmState(1, mtot, state.rho)
    dstate.load(0, state)
    dx, du, dstats = solve_batched(ctx, dqp, settings, dstate)
    K, k, P, p = export_solution(ctx)
    dstate.store(0, state)
    stats = AdmmStats(iterations=int(dstats.iterations[0]), converged=bool(dstats.converged[0]),
                      r_primal=state.r_primal, r_dual=state.r_dual, rho=state.rho,
                      rho_changes=int(dstats.rho_changes[0]), cache_builds=int(dstats.cache_builds[0]),
                      scan_layers=scan_depth(N + 1))
    sol = lqr.LqrSolution(dx=to_host(dx[0]), du=to_host(du[0]), K=to_host(K[0]), k=to_host(k[0]),
                          P=to_host(P[0]), p=to_host(p[0]), scan_layers=stats.scan_layers)
    return AdmmResult(dx=sol.dx, du=sol.du, state=state, stats=stats, solution=sol)
