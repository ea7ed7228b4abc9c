"""Drop-in for ``scanmpc.sls``: SLS synthesis, tube tightening and the robust loops on the GPU.

Same names, dataclasses and signatures as /root/reference/pkg/src/scanmpc/sls.py:
``SlsWeights`` (:33-48), ``SlsResponse`` (:51-92, ragged ``[j][k-j-1]``),
``SlsDuals`` (:95-111), ``Tightening`` (:114-126), ``SlsCosts`` (:129-143),
``row_norms`` (:146), ``compute_duals`` (:150), ``assemble_costs`` (:176),
``synthesize`` (:227), ``tighten`` (:329), ``sls_cost`` (:344),
``RobustSettings`` / ``RobustStats`` / ``RobustResult`` (:361-390),
``solve_robust`` (:400), ``RobustRtiResult`` / ``rti_robust_step`` (:487-525).

All arithmetic runs in csrc/sls.cu (triangular cell layout, column-batched
scans with neutral elements elided).  Objects returned here carry a token of
the device workspace that produced them, so chaining calls (assemble ->
synthesize -> tighten -> compute_duals) does not round-trip through the host.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from . import sqp
from .device import Context, resolve, stream_ptr, to_dev, to_host
from .engine import RtiEngine, alloc_qp
from .errors import RobustInfeasibleError, SingularStageError  # noqa: F401

F32, F64 = torch.float32, torch.float64


# --- dataclasses (sls.py:33-143) -----------------------------------------------------

@dataclass
class SlsWeights:
    Qbar: np.ndarray
    Rbar: np.ndarray
    QbarN: np.ndarray

    @classmethod
    def identity(cls, nx: int, nu: int, scale: float = 1.0) -> "SlsWeights":
        return cls(scale * np.eye(nx), scale * np.eye(nu), scale * np.eye(nx))

    def validate(self):
        for name in ("Qbar", "Rbar", "QbarN"):
            M = np.asarray(getattr(self, name))
            if not np.allclose(M, M.T):
                raise ValueError(f"{name} must be symmetric")
            np.linalg.cholesky(M)


@dataclass
class SlsResponse:
    Phi_x: list
    Phi_u: list
    gains: list
    N: int
    nx: int
    nu: int

    def phi_x(self, k: int, j: int) -> np.ndarray:
        return self.Phi_x[j][k - j - 1]

    def phi_u(self, k: int, j: int) -> np.ndarray:
        return self.Phi_u[j][k - j - 1]

    def scaled(self, factor: float) -> "SlsResponse":
        return SlsResponse([factor * p for p in self.Phi_x], [factor * p for p in self.Phi_u],
                           [g.copy() for g in self.gains], self.N, self.nx, self.nu)

    @classmethod
    def zero(cls, N: int, nx: int, nu: int) -> "SlsResponse":
        return cls(Phi_x=[np.zeros((N - j, nx, nx)) for j in range(N)],
                   Phi_u=[np.zeros((max(N - 1 - j, 0), nu, nx)) for j in range(N)],
                   gains=[np.zeros((max(N - 1 - j, 0), nu, nx)) for j in range(N)], N=N, nx=nx, nu=nu)

    def dynamics_residual(self, A, B) -> float:
        worst = 0.0
        for j in range(self.N):
            for k in range(j + 1, self.N):
                pred = A[k] @ self.phi_x(k, j) + B[k] @ self.phi_u(k, j)
                worst = max(worst, float(np.abs(self.phi_x(k + 1, j) - pred).max()))
        return worst


class DeviceSlsResponse(SlsResponse):
    """An SlsResponse whose blocks stay on the device until first accessed."""

    def __init__(self, phix, phiu, gains, N, nx, nu, token=None):
        self._cells = (phix, phiu, gains)
        self._host = None
        self.N, self.nx, self.nu = N, nx, nu
        self._tok = token

    def _materialize(self):
        if self._host is None:
            px, pu, g = (to_host(t) for t in self._cells)
            self._host = (cells_to_ragged(px, self.N, 1, self.N + 1), cells_to_ragged(pu, self.N, 1, self.N),
                          cells_to_ragged(g, self.N, 1, self.N))
        return self._host

    Phi_x = property(lambda self: self._materialize()[0])
    Phi_u = property(lambda self: self._materialize()[1])
    gains = property(lambda self: self._materialize()[2])


@dataclass
class SlsDuals:
    tau: list
    tau_term: np.ndarray
    beta: list
    beta_term: np.ndarray
    eps: float

    @classmethod
    def zero(cls, N: int, nc: int, nf: int, eps: float = 1e-8) -> "SlsDuals":
        return cls(tau=[np.zeros((max(N - 1 - j, 0), nc)) for j in range(N)], tau_term=np.zeros((N, nf)),
                   beta=[np.zeros((max(N - 1 - j, 0), nc)) for j in range(N)], beta_term=np.zeros((N, nf)),
                   eps=eps)


@dataclass
class Tightening:
    h: np.ndarray
    hf: np.ndarray

    @classmethod
    def zero(cls, N: int, nc: int, nf: int) -> "Tightening":
        return cls(h=np.zeros((N, nc)), hf=np.zeros(nf))

    def max_abs_diff(self, other: "Tightening") -> float:
        return max(float(np.abs(self.h - other.h).max(initial=0.0)),
                   float(np.abs(self.hf - other.hf).max(initial=0.0)))


@dataclass
class SlsCosts:
    Qx: list
    Qu: list
    Qux: list
    Qx_term: np.ndarray

    def blocks(self, k: int, j: int):
        i = k - j - 1
        return self.Qx[j][i], self.Qu[j][i], self.Qux[j][i]

    def terminal(self, j: int) -> np.ndarray:
        return self.Qx_term[j]


def row_norms(M) -> np.ndarray:
    """sls.py:146-147 (host helper)."""
    return np.sqrt((np.asarray(M) * np.asarray(M)).sum(axis=-1))


# --- triangular cell layout (include/gsls.h) -------------------------------------------

def cell_index(N: int, k: int, j: int) -> int:
    return j * N - j * (j - 1) // 2 + (k - j - 1)


def ragged_to_cells(ragged, N: int, shape, terminal=None) -> np.ndarray:
    """ragged[j][k-j-1] (k from j+1) -> (ncell, *shape); ``terminal[j]`` -> cell (N, j)."""
    out = np.zeros((N * (N + 1) // 2,) + tuple(shape))
    for j in range(N):
        o = cell_index(N, j + 1, j)
        blk = np.asarray(ragged[j]) if ragged is not None else np.zeros((0,) + tuple(shape))
        out[o:o + len(blk)] = blk
        if terminal is not None:
            out[cell_index(N, N, j)] = terminal[j]
    return out


def cells_to_ragged(cells, N: int, start: int, stop: int) -> list:
    """(ncell, ...) -> [j] -> array over k in [j+start, stop)."""
    return [np.ascontiguousarray(cells[cell_index(N, j + start, j): cell_index(N, j + start, j) + max(stop - j - start, 0)])
            for j in range(N)]


# --- device workspace ------------------------------------------------------------------

class _Ws:
    """Batch-1 SLS workspace for one (n, m, c, nf, N)."""

    def __init__(self, n, m, c, nf, N):
        self.dims = (n, m, c, nf, N)
        self.ctx = Context(n, m, c, nf, N, 1)
        self.qp = alloc_qp(1, n, m, c, nf, N)
        self.E = torch.zeros(1, N, n, n, dtype=F32, device=self.qp.QN.device)
        self.ncell = N * (N + 1) // 2
        self.version = 0    # bumped whenever the held costs / response change
        self.costs_ver = -1
        self.resp_ver = -1

    def bump(self):
        self.version += 1
        return self.version


def _ws(n, m, c, nf, N, executor=None, columns=None) -> _Ws:
    dev = resolve(executor)
    cache = dev.__dict__.setdefault("_sls_ws", {})
    key = (n, m, c, nf, N) + ((tuple(columns),) if columns is not None else ())
    if key not in cache:
        ws = _Ws(n, m, c, nf, N)
        if columns is not None:  # column shard: every SLS array holds only the shard's cells
            j0, j1 = columns
            nat.check(ws.ctx.lib.gsls_sls_set_columns(ws.ctx.handle, j0, j1), "sls columns")
            ws.columns = (j0, j1)
            ws.cell0 = cell_index(N, j0 + 1, j0)
            ws.ncell = cell_index(N, j1 + 1, j1) - ws.cell0
        cache[key] = ws
    return cache[key]


def _set_constraints(ws: _Ws, C, D, CN):
    ws.qp.C.copy_(to_dev(C, F32)[None])
    ws.qp.D.copy_(to_dev(D, F32)[None])
    ws.qp.CN.copy_(to_dev(CN, F32)[None])


def _ensure_response(ws: _Ws, response):
    tok = getattr(response, "_tok", None)
    if tok is not None and tok[0] is ws and tok[1] == ws.resp_ver:
        return
    n, m, c, nf, N = ws.dims
    phix = to_dev(ragged_to_cells(response.Phi_x, N, (n, n)), F32)[None].contiguous()
    phiu = to_dev(ragged_to_cells(response.Phi_u, N, (m, n)), F32)[None].contiguous()
    nat.check(ws.ctx.lib.gsls_sls_import_response(ws.ctx.handle, phix.data_ptr(), phiu.data_ptr(), stream_ptr()),
              "import response")
    ws.resp_ver = ws.bump()
    response._tok = (ws, ws.resp_ver)


def _duals_from_cells(tau, tau_term, beta, beta_term, N, eps) -> SlsDuals:
    return SlsDuals(tau=cells_to_ragged(tau, N, 1, N), tau_term=tau_term,
                    beta=cells_to_ragged(beta, N, 1, N), beta_term=beta_term, eps=eps)


# --- entry points ----------------------------------------------------------------------

def compute_duals(lam_stage, lam_term, response, C, D, CN, eps: float = 1e-8, executor=None) -> SlsDuals:
    """tau = max(lam, 0) / sqrt(beta + eps), beta = squared constraint-mapped row norms (sls.py:150-173)."""
    lam_stage, lam_term = np.asarray(lam_stage, float), np.asarray(lam_term, float)
    N, c = lam_stage.shape
    nf = lam_term.shape[0]
    C, D, CN = np.asarray(C, float), np.asarray(D, float), np.asarray(CN, float)
    n, m = C.shape[2], D.shape[2]
    ws = _ws(n, m, c, nf, N, executor)
    _set_constraints(ws, C, D, CN)
    use = response is not None
    if use:
        _ensure_response(ws, response)
    lam = to_dev(np.concatenate([lam_stage.ravel(), lam_term]), F64)[None].contiguous()
    dev = lam.device
    tau = torch.zeros(1, ws.ncell, c, dtype=F64, device=dev)
    beta = torch.zeros_like(tau)
    tt = torch.zeros(1, N, nf, dtype=F64, device=dev)
    bt = torch.zeros_like(tt)
    s = ws.qp.cstruct()
    nat.check(ws.ctx.lib.gsls_sls_duals(ws.ctx.handle, ctypes.byref(s), lam.data_ptr(), float(eps), int(use), 0,
                                        tau.data_ptr() if tau.numel() else None,
                                        tt.data_ptr() if tt.numel() else None,
                                        beta.data_ptr() if beta.numel() else None,
                                        bt.data_ptr() if bt.numel() else None, stream_ptr()), "compute_duals")
    return _duals_from_cells(to_host(tau[0]), to_host(tt[0]), to_host(beta[0]), to_host(bt[0]), N, eps)


def assemble_costs(duals: SlsDuals | None, C, D, CN, weights: SlsWeights, executor=None) -> SlsCosts:
    """Cost blocks [C D]' diag(tau) [C D] + blkdiag(Qbar, Rbar) per (k, j) (sls.py:176-200)."""
    C, D, CN = np.asarray(C, float), np.asarray(D, float), np.asarray(CN, float)
    N, c, n = C.shape
    m, nf = D.shape[2], CN.shape[0]
    ws = _ws(n, m, c, nf, N, executor)
    _set_constraints(ws, C, D, CN)
    tau = tt = None
    if duals is not None:
        tau = to_dev(ragged_to_cells(duals.tau, N, (c,)), F64)[None].contiguous()
        tt = to_dev(np.asarray(duals.tau_term, float).reshape(N, nf), F64)[None].contiguous()
    W = [to_dev(np.asarray(a, float), F32) for a in (weights.Qbar, weights.Rbar, weights.QbarN)]
    s = ws.qp.cstruct()
    lib, h, S = ws.ctx.lib, ws.ctx.handle, stream_ptr()
    nat.check(lib.gsls_sls_assemble(h, ctypes.byref(s), tau.data_ptr() if tau is not None and tau.numel() else None,
                                    tt.data_ptr() if tt is not None and tt.numel() else None,
                                    W[0].data_ptr(), W[1].data_ptr(), W[2].data_ptr(), 0, S), "assemble_costs")
    dev = ws.qp.QN.device
    Qx = torch.empty(1, ws.ncell, n, n, dtype=F64, device=dev)
    Qu = torch.empty(1, ws.ncell, m, m, dtype=F64, device=dev)
    Qux = torch.empty(1, ws.ncell, m, n, dtype=F64, device=dev)
    nat.check(lib.gsls_sls_export_costs(h, Qx.data_ptr(), Qu.data_ptr(), Qux.data_ptr(), S), "export costs")
    ws.costs_ver = ws.bump()
    qx, qu, qux = to_host(Qx[0]), to_host(Qu[0]), to_host(Qux[0])
    costs = SlsCosts(Qx=cells_to_ragged(qx, N, 1, N), Qu=cells_to_ragged(qu, N, 1, N),
                     Qux=cells_to_ragged(qux, N, 1, N),
                     Qx_term=np.stack([qx[cell_index(N, N, j)] for j in range(N)]) if N else np.zeros((0, n, n)))
    costs._tok = (ws, ws.costs_ver)
    return costs


def synthesize(A, B, E, costs: SlsCosts, executor=None) -> SlsResponse:
    """All per-disturbance Riccati problems by one batched scan pair (sls.py:227-318)."""
    A, B, E = np.asarray(A, float), np.asarray(B, float), np.asarray(E, float)
    N, n, m = A.shape[0], A.shape[-1], B.shape[-1]
    if N == 0:
        return SlsResponse.zero(0, n, m)
    tok = getattr(costs, "_tok", None)
    if tok is not None and tok[1] == tok[0].costs_ver and tok[0].dims[0] == n and tok[0].dims[4] == N:
        ws = tok[0]
    else:
        ws = _ws(n, m, 0, 0, N, executor)
        Qx = to_dev(ragged_to_cells(costs.Qx, N, (n, n), terminal=costs.Qx_term), F64)[None].contiguous()
        Qu = to_dev(ragged_to_cells(costs.Qu, N, (m, m)), F64)[None].contiguous()
        Qux = to_dev(ragged_to_cells(costs.Qux, N, (m, n)), F64)[None].contiguous()
        nat.check(ws.ctx.lib.gsls_sls_set_costs(ws.ctx.handle, Qx.data_ptr(), Qu.data_ptr(), Qux.data_ptr(),
                                                stream_ptr()), "set costs")
        ws.costs_ver = ws.bump()
    ws.qp.A.copy_(to_dev(A, F32)[None])
    ws.qp.B.copy_(to_dev(B, F32)[None])
    ws.E.copy_(to_dev(E, F32)[None])
    s = ws.qp.cstruct()
    nat.check(ws.ctx.lib.gsls_sls_synthesize(ws.ctx.handle, ctypes.byref(s), ws.E.data_ptr(), stream_ptr()),
              "synthesize")
    ws.resp_ver = ws.bump()
    return _export_response(ws)


def _export_response(ws: _Ws) -> DeviceSlsResponse:
    n, m, c, nf, N = ws.dims
    dev = ws.qp.QN.device
    phix = torch.empty(ws.ncell, n, n, dtype=F32, device=dev)
    phiu = torch.empty(ws.ncell, m, n, dtype=F32, device=dev)
    gains = torch.empty_like(phiu)
    nat.check(ws.ctx.lib.gsls_sls_export(ws.ctx.handle, phix.data_ptr(), phiu.data_ptr(), gains.data_ptr(),
                                         stream_ptr()), "export response")
    return DeviceSlsResponse(phix, phiu, gains, N, n, m, token=(ws, ws.resp_ver))


def tighten(response: SlsResponse, C, D, CN, executor=None) -> Tightening:
    """h_k = sum_{j<k} rownorm(C_k Phi^x_{k,j} + D_k Phi^u_{k,j}); terminal analog (sls.py:329-341)."""
    C, D, CN = np.asarray(C, float), np.asarray(D, float), np.asarray(CN, float)
    N, c, n = C.shape
    m, nf = D.shape[2], CN.shape[0]
    ws = _ws(n, m, c, nf, N, executor)
    _set_constraints(ws, C, D, CN)
    _ensure_response(ws, response)
    dev = ws.qp.QN.device
    h = torch.zeros(1, N, c, dtype=F64, device=dev)
    hf = torch.zeros(1, nf, dtype=F64, device=dev)
    s = ws.qp.cstruct()
    nat.check(ws.ctx.lib.gsls_sls_tighten(ws.ctx.handle, ctypes.byref(s), h.data_ptr() if h.numel() else None,
                                          hf.data_ptr() if hf.numel() else None, stream_ptr()), "tighten")
    return Tightening(h=to_host(h[0]), hf=to_host(hf[0]))


def synthesize_tighten_columns(A, B, E, costs: SlsCosts, C, D, CN, columns, executor=None):
    """One column shard of synthesize + tighten: the disturbance
    columns j in ``columns = (j0, j1)`` only (sls.py:227-341; columns are independent).

    Returns (h_part, hf_part, phix, phiu): the shard's partial sums of the stage /
    terminal tightening (sum them over shards) and its response cells, shard-local
    (cell(k, j) - cell(j0 + 1, j0)), float32 device tensors."""
    A, B, E = np.asarray(A, float), np.asarray(B, float), np.asarray(E, float)
    C, D, CN = np.asarray(C, float), np.asarray(D, float), np.asarray(CN, float)
    N, n, m = A.shape[0], A.shape[-1], B.shape[-1]
    c, nf = C.shape[1], CN.shape[0]
    ws = _ws(n, m, c, nf, N, executor, columns=columns)
    sl = slice(ws.cell0, ws.cell0 + ws.ncell)
    Qx = to_dev(ragged_to_cells(costs.Qx, N, (n, n), terminal=costs.Qx_term)[sl], F64)[None].contiguous()
    Qu = to_dev(ragged_to_cells(costs.Qu, N, (m, m))[sl], F64)[None].contiguous()
    Qux = to_dev(ragged_to_cells(costs.Qux, N, (m, n))[sl], F64)[None].contiguous()
    lib, hd = ws.ctx.lib, ws.ctx.handle
    nat.check(lib.gsls_sls_set_costs(hd, Qx.data_ptr(), Qu.data_ptr(), Qux.data_ptr(), stream_ptr()), "set costs")
    ws.qp.A.copy_(to_dev(A, F32)[None])
    ws.qp.B.copy_(to_dev(B, F32)[None])
    ws.E.copy_(to_dev(E, F32)[None])
    _set_constraints(ws, C, D, CN)
    st = ws.qp.cstruct()
    nat.check(lib.gsls_sls_synthesize(hd, ctypes.byref(st), ws.E.data_ptr(), stream_ptr()), "synthesize")
    dev = ws.qp.QN.device
    h = torch.zeros(1, N, c, dtype=F64, device=dev)
    hf = torch.zeros(1, nf, dtype=F64, device=dev)
    nat.check(lib.gsls_sls_tighten(hd, ctypes.byref(st), h.data_ptr() if h.numel() else None,
                                   hf.data_ptr() if hf.numel() else None, stream_ptr()), "tighten")
    phix = torch.empty(ws.ncell, n, n, dtype=F32, device=dev)
    phiu = torch.empty(ws.ncell, m, n, dtype=F32, device=dev)
    nat.check(lib.gsls_sls_export(hd, phix.data_ptr(), phiu.data_ptr(), None, stream_ptr()), "export response")
    ws.resp_ver = ws.bump()
    return h[0], hf[0], phix, phiu


def sls_cost(response: SlsResponse, weights: SlsWeights, executor=None) -> float:
    """Weighted Frobenius energy of the response maps (sls.py:344-358), computed by
    gsls_sls_cost on the device response (a host response is loaded first): the sum over
    cells of ||L' Phi||_F^2 = tr(Phi' W Phi).  The weights must be positive definite, as
    the reference's Cholesky factors require (np.linalg.LinAlgError otherwise)."""
    W = [np.asarray(w, float) for w in (weights.Qbar, weights.Rbar, weights.QbarN)]
    for w in W:
        np.linalg.cholesky(w)  # the reference's factorization: same error on an indefinite weight
    N, nx, nu = response.N, response.nx, response.nu
    if N == 0:
        return 0.0
    tok = getattr(response, "_tok", None)
    ws = tok[0] if tok is not None and tok[1] == tok[0].resp_ver else _ws(nx, nu, 1, 1, N, executor)
    _ensure_response(ws, response)
    Qb, Rb, QbN = (to_dev(w, F64).contiguous() for w in W)
    out = torch.zeros(1, dtype=F64, device=Qb.device)
    nat.check(ws.ctx.lib.gsls_sls_cost(ws.ctx.handle, Qb.data_ptr(), Rb.data_ptr(), QbN.data_ptr(), out.data_ptr(),
                                       stream_ptr()), "sls_cost")
    return float(out[0])


# --- robust loops ------------------------------------------------------------------------

@dataclass
class RobustSettings:
    sqp: sqp.SqpSettings = field(default_factory=sqp.SqpSettings)
    weights: SlsWeights | None = None
    eps: float = 1e-8
    tol_h: float = 1e-3
    max_alternations: int = 20
    weight_scale: float = 1.0
    tau_damping: float = 0.5


@dataclass
class RobustStats:
    alternations: int = 0
    converged: bool = False
    dh: float = np.inf
    sqp_iterations: int = 0
    nominal_converged: bool = True


@dataclass
class RobustResult:
    trajectory: sqp.Trajectory
    response: SlsResponse
    tightening: Tightening
    duals: SlsDuals
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: RobustStats
    qp: object


@dataclass
class RobustRtiResult:
    u0: np.ndarray
    warm_start: sqp.Trajectory
    plan: sqp.Trajectory
    tau: SlsDuals
    tightening: Tightening
    response: SlsResponse
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: sqp.SqpStats


def _stage_disturbances(model, traj, inflation=None) -> np.ndarray:
    """sls.py:393-397."""
    E = np.stack([model.disturbance(traj.x[k]) for k in range(traj.N)])
    if inflation is not None:
        E = E + np.stack([inflation(k, traj.x[k]) for k in range(traj.N)])
    return E


def _blend_duals(fresh: SlsDuals, previous: SlsDuals | None, damping: float) -> SlsDuals:
    """sls.py:476-484."""
    if previous is None or damping <= 0.0:
        return fresh
    keep = damping
    for j in range(len(fresh.tau)):
        if fresh.tau[j].size:
            fresh.tau[j] = (1 - keep) * fresh.tau[j] + keep * previous.tau[j]
    fresh.tau_term = (1 - keep) * fresh.tau_term + keep * previous.tau_term
    return fresh


def _weights(model, settings: RobustSettings) -> SlsWeights:
    return settings.weights or SlsWeights.identity(model.nx, model.nu, settings.weight_scale)


def solve_robust(model, x_bar0, settings: RobustSettings, initial=None, executor=None,
                 e_inflation=None) -> RobustResult:
    """Alternate tightened nominal solves with controller synthesis (sls.py:400-469)."""
    x_bar0 = np.asarray(x_bar0, float)
    weights = _weights(model, settings)
    guess, tight, response, duals = initial, None, None, None
    stats = RobustStats()
    infeasible_run = 0
    result = None
    last_good = None
    for alt in range(settings.max_alternations + 1):
        try:
            nominal = sqp.solve_nmpc(model, x_bar0, settings.sqp,
                                     guess if guess is not None else sqp.initial_guess(model, x_bar0, 32),
                                     tightenings=tight, executor=executor)
        except sqp.DivergenceError:
            if last_good is None:
                raise
            nominal = None
        if nominal is None or not nominal.stats.converged:
            infeasible_run += 1
            if infeasible_run >= 3:
                raise RobustInfeasibleError("robust problem infeasible: reduce disturbance or relax constraints")
            if nominal is None:
                nominal = last_good
        else:
            infeasible_run = 0
            last_good = nominal
        stats.sqp_iterations += nominal.stats.iterations
        stats.nominal_converged = nominal.stats.converged and infeasible_run == 0
        guess = nominal.trajectory
        qp = sqp.linearize(model, nominal.trajectory, tight, x_bar0, executor=executor)
        if response is not None:
            result = RobustResult(trajectory=nominal.trajectory, response=response, tightening=tight,
                                  duals=duals or SlsDuals.zero(qp.N, qp.nc, qp.nf, settings.eps),
                                  lam_stage=nominal.lam_stage, lam_terminal=nominal.lam_terminal, stats=stats,
                                  qp=qp)
            if stats.dh <= settings.tol_h:
                stats.converged = True
                break
        if alt == settings.max_alternations:
            break
        stats.alternations = alt + 1
        if response is None:
            duals = None
        else:
            fresh = compute_duals(nominal.lam_stage, nominal.lam_terminal, response, qp.C, qp.D, qp.CN,
                                  settings.eps, executor=executor)
            duals = _blend_duals(fresh, duals, settings.tau_damping)
        costs = assemble_costs(duals, qp.C, qp.D, qp.CN, weights, executor=executor)
        E = _stage_disturbances(model, nominal.trajectory, e_inflation)
        response = synthesize(qp.A, qp.B, E, costs, executor=executor)
        new_tight = tighten(response, qp.C, qp.D, qp.CN, executor=executor)
        stats.dh = (new_tight.max_abs_diff(tight)
                    if tight is not None and tight.h.shape == new_tight.h.shape else np.inf)
        tight = new_tight
    return result


def _engine(model, N: int, settings: RobustSettings, executor=None) -> RtiEngine:
    dev = resolve(executor)
    cache = dev.__dict__.setdefault("_rti_engines", {})
    key = (id(model), N, id(settings))
    eng = cache.get(key)
    if eng is None or eng.model is not model or eng.settings is not settings:
        eng = RtiEngine(model, N, 1, settings, robust=True)
        cache[key] = eng
    return eng


def rti_robust_step(model, x_bar0, previous: sqp.Trajectory, tau: SlsDuals | None, settings: RobustSettings,
                    executor=None, e_inflation=None, warm_admm=None) -> RobustRtiResult:
    """One linearization, one controller update, one tightened nominal update (sls.py:500-525)."""
    N = previous.N
    eng = _engine(model, N, settings, executor)
    n, m, c, nf, _ = eng.dims
    xb = to_dev(np.asarray(x_bar0, float), F64)[None].contiguous()
    px = to_dev(previous.x, F64)[None].contiguous()
    pu = to_dev(previous.u, F64)[None].contiguous()
    t_cells = tt = None
    if tau is not None:
        t_cells = to_dev(ragged_to_cells(tau.tau, N, (c,)), F64)[None]
        tt = to_dev(np.asarray(tau.tau_term, float).reshape(N, nf), F64)[None]
    E = None
    if e_inflation is not None:
        E = to_dev(_stage_disturbances(model, previous, e_inflation), F32)[None]
    if warm_admm is not None:
        eng.state.load(0, warm_admm)
    eng.step(xb, px, pu, tau=t_cells, tau_term=tt, use_tau=tau is not None, E=E, warm_admm=warm_admm is not None)
    if warm_admm is not None:
        eng.state.store(0, warm_admm)
    lam_s, lam_t = eng.lam_split()
    phix, phiu, gains = eng.export_response()
    resp = DeviceSlsResponse(phix[0], phiu[0], gains[0], N, n, m)
    tau_next = SlsDuals(tau=cells_to_ragged(to_host(eng.tau[0]), N, 1, N), tau_term=to_host(eng.tau_term[0]),
                        beta=cells_to_ragged(to_host(eng.beta[0]), N, 1, N), beta_term=to_host(eng.beta_term[0]),
                        eps=settings.eps)
    conv = bool(eng.stats.converged[0])
    r_p, r_d = float(eng.state.r_primal[0]), float(eng.state.r_dual[0])
    stats = sqp.SqpStats(iterations=1, converged=conv, residual=max(r_p, r_d),
                         admm_iterations=int(eng.stats.iterations[0]), scan_layers=2 * (N + 1 - 1).bit_length(),
                         admm_converged=conv, cost=float(eng.cost[0]))
    plan = sqp.Trajectory(to_host(eng.plan_x[0]), to_host(eng.plan_u[0]), previous.dt)
    warm = sqp.Trajectory(to_host(eng.warm_x[0]), to_host(eng.warm_u[0]), previous.dt)
    return RobustRtiResult(u0=to_host(eng.u0[0]), warm_start=warm, plan=plan, tau=tau_next,
                           tightening=Tightening(to_host(eng.h[0]), to_host(eng.hf[0])), response=resp,
                           lam_stage=to_host(lam_s[0]), lam_terminal=to_host(lam_t[0]), stats=stats)
