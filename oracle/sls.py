"""Oracle (test infrastructure): SLS synthesis, tightening and the robust loops.

Restates /root/reference/pkg/src/scanmpc/sls.py in float64 numpy:
ragged response storage [j][k-j-1] (sls.py:51-92), duals tau = lam/sqrt(beta+eps)
(sls.py:150-173), cost blocks (sls.py:176-200), the grid CVF reverse scan with
neutral elements plus the forward product scan (sls.py:203-318), tube
tightening (sls.py:329-341), the weighted energy (sls.py:344-358), the batch
alternation (sls.py:400-484) and the RTI robust step (sls.py:500-525).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import lqr, sqp, tree


class RobustInfeasibleError(RuntimeError):
    pass


@dataclass
class Weights:
    Qbar: np.ndarray
    Rbar: np.ndarray
    QbarN: np.ndarray

    @classmethod
    def identity(cls, nx, nu, scale=1.0):
        return cls(scale * np.eye(nx), scale * np.eye(nu), scale * np.eye(nx))


@dataclass
class Response:
    Phi_x: list
    Phi_u: list
    gains: list
    N: int
    nx: int
    nu: int

    def phi_x(self, k, j):
        return self.Phi_x[j][k - j - 1]

    def phi_u(self, k, j):
        return self.Phi_u[j][k - j - 1]


@dataclass
class Duals:
    tau: list
    tau_term: np.ndarray
    beta: list
    beta_term: np.ndarray
    eps: float

    @classmethod
    def zero(cls, N, nc, nf, eps=1e-8):
        return cls([np.zeros((max(N - 1 - j, 0), nc)) for j in range(N)], np.zeros((N, nf)),
                   [np.zeros((max(N - 1 - j, 0), nc)) for j in range(N)], np.zeros((N, nf)), eps)


@dataclass
class Tightening:
    h: np.ndarray
    hf: np.ndarray

    def max_abs_diff(self, other):
        return max(float(np.abs(self.h - other.h).max(initial=0.0)),
                   float(np.abs(self.hf - other.hf).max(initial=0.0)))


@dataclass
class Costs:
    Qx: list
    Qu: list
    Qux: list
    Qx_term: np.ndarray


def row_norms(M):
    return np.sqrt((M * M).sum(axis=-1))


def compute_duals(lam_stage, lam_term, resp, C, D, CN, eps=1e-8):
    """sls.py:150-173."""
    N, nc = lam_stage.shape
    nf = lam_term.shape[0]
    ls = np.clip(lam_stage, 0.0, None)
    lt = np.clip(lam_term, 0.0, None)
    out = Duals.zero(N, nc, nf, eps)
    for j in range(N):
        for k in range(j + 1, N):
            if resp is not None:
                out.beta[j][k - j - 1] = row_norms(C[k] @ resp.phi_x(k, j) + D[k] @ resp.phi_u(k, j)) ** 2
            out.tau[j][k - j - 1] = ls[k] / np.sqrt(out.beta[j][k - j - 1] + eps)
        if resp is not None and nf:
            out.beta_term[j] = row_norms(CN @ resp.phi_x(N, j)) ** 2
        out.tau_term[j] = lt / np.sqrt(out.beta_term[j] + eps)
    return out


def assemble_costs(duals, C, D, CN, w: Weights) -> Costs:
    """sls.py:176-200."""
    N = C.shape[0]
    nx, nu = w.Qbar.shape[0], w.Rbar.shape[0]
    Qx, Qu, Qux = [], [], []
    Qt = np.empty((N, nx, nx))
    for j in range(N):
        cnt = max(N - 1 - j, 0)
        a = np.empty((cnt, nx, nx)); b = np.empty((cnt, nu, nu)); c = np.empty((cnt, nu, nx))
        for k in range(j + 1, N):
            t = duals.tau[j][k - j - 1] if duals is not None else np.zeros(C.shape[1])
            CtT, DtT = C[k].T * t, D[k].T * t
            a[k - j - 1] = CtT @ C[k] + w.Qbar
            b[k - j - 1] = DtT @ D[k] + w.Rbar
            c[k - j - 1] = DtT @ C[k]
        Qx.append(a); Qu.append(b); Qux.append(c)
        tN = duals.tau_term[j] if duals is not None else np.zeros(CN.shape[0])
        Qt[j] = (CN.T * tN) @ CN + w.QbarN
    return Costs(Qx, Qu, Qux, Qt)


def _grid_cvf(lhs, rhs):
    P, A, C, _, _ = lqr.cvf_matrix(lhs[0], lhs[1], lhs[2], rhs[0], rhs[1], rhs[2])
    return (P, A, C), ()


def _grid_unit(k, J, n):
    I = np.zeros((k, J, n, n))
    I[...] = np.eye(n)
    return (np.zeros((k, J, n, n)), I, np.zeros((k, J, n, n)))


def _matprod(lhs, rhs):
    return (rhs[0] @ lhs[0],), ()


def _locate(grid, valid, label):
    for (k, j) in np.argwhere(valid):
        try:
            np.linalg.cholesky(grid[k, j])
        except np.linalg.LinAlgError:
            raise lqr.SingularStageError(f"singular {label} block at (k={k}, j={j})") from None


def synthesize(A, B, E, costs: Costs) -> Response:
    """All per-disturbance Riccati problems via one grid scan pair (sls.py:227-318)."""
    A = np.asarray(A, float); B = np.asarray(B, float); E = np.asarray(E, float)
    N, nx, nu = A.shape[0], A.shape[-1], B.shape[-1]
    if N == 0:
        return Response([], [], [], 0, nx, nu)
    Qx = np.tile(np.eye(nx), (N, N, 1, 1))
    Qu = np.tile(np.eye(nu), (N, N, 1, 1))
    Qux = np.zeros((N, N, nu, nx))
    valid = np.zeros((N, N), bool)
    for j in range(N):
        for k in range(j + 1, N):
            Qx[k, j], Qu[k, j], Qux[k, j] = costs.Qx[j][k - j - 1], costs.Qu[j][k - j - 1], costs.Qux[j][k - j - 1]
            valid[k, j] = True
    try:
        Qui = lqr.spd_inverse(Qu, "synthesis input-cost block")
    except lqr.SingularStageError:
        _locate(Qu, valid, "Qu")
        raise
    Ag = np.broadcast_to(A[:, None], (N, N, nx, nx))
    Bg = np.broadcast_to(B[:, None], (N, N, nx, nu))
    BgT = np.swapaxes(Bg, -1, -2)
    QQ = Qui @ Qux
    Pel = np.ascontiguousarray(Qx - np.swapaxes(Qux, -1, -2) @ QQ)
    Ael = np.ascontiguousarray(Ag - Bg @ QQ)
    Cel = np.ascontiguousarray(Bg @ Qui @ BgT)
    off = ~valid
    Pel[off] = 0.0
    Ael[off] = np.eye(nx)
    Cel[off] = 0.0
    elems = (np.concatenate([Pel, costs.Qx_term[None]]),
             np.concatenate([Ael, np.zeros((1, N, nx, nx))]),
             np.concatenate([Cel, np.zeros((1, N, nx, nx))]))
    out, _ = tree.scan(elems, _grid_cvf, lambda c: _grid_unit(c, N, nx), reverse=True)
    Pn = np.ascontiguousarray(out[0][1:])
    inner = Qu + BgT @ Pn @ Bg
    try:
        G = lqr.spd_inverse(inner, "synthesis innovation")
    except lqr.SingularStageError:
        _locate(inner, valid, "Qu + B'PB")
        raise
    K = -(G @ (Qux + BgT @ Pn @ Ag))
    M = np.tile(np.eye(nx), (N, N, 1, 1))
    d = np.arange(N)
    M[d, d] = E
    cl = Ag + Bg @ K
    M[valid] = cl[valid]
    prod, _ = tree.scan((np.ascontiguousarray(M),), _matprod, lambda c: (_grid_unit(c, N, nx)[1],))
    Phi = prod[0]
    Px, Pu, gains = [], [], []
    for j in range(N):
        px = np.ascontiguousarray(Phi[j:, j])
        kj = np.ascontiguousarray(K[j + 1:, j])
        Px.append(px)
        Pu.append(kj @ px[:-1] if N - 1 - j > 0 else np.zeros((0, nu, nx)))
        gains.append(kj)
    return Response(Px, Pu, gains, N, nx, nu)


def tighten(resp: Response, C, D, CN) -> Tightening:
    """sls.py:329-341."""
    N = resp.N
    nc, nf = C.shape[1], CN.shape[0]
    h = np.zeros((N, nc))
    for k in range(1, N):
        for j in range(k):
            h[k] += row_norms(C[k] @ resp.phi_x(k, j) + D[k] @ resp.phi_u(k, j))
    hf = np.zeros(nf)
    if nf:
        for j in range(N):
            hf += row_norms(CN @ resp.phi_x(N, j))
    return Tightening(h, hf)


def sls_cost(resp: Response, w: Weights) -> float:
    """sls.py:344-358."""
    Lq, Lr, Ln = (np.linalg.cholesky(w.Qbar), np.linalg.cholesky(w.Rbar), np.linalg.cholesky(w.QbarN))
    tot = 0.0
    for j in range(resp.N):
        px = resp.Phi_x[j]
        if px.shape[0] > 1:
            tot += float(((Lq.T @ px[:-1]) ** 2).sum())
        tot += float(((Ln.T @ px[-1]) ** 2).sum())
        if resp.Phi_u[j].shape[0]:
            tot += float(((Lr.T @ resp.Phi_u[j]) ** 2).sum())
    return tot


def fastsls_sequential(A, B, E, costs: Costs) -> Response:
    """Per-column Riccati + forward propagation by direct loops (reference.py:65-95)."""
    A = np.asarray(A, float); B = np.asarray(B, float); E = np.asarray(E, float)
    N, nx, nu = A.shape[0], A.shape[-1], B.shape[-1]
    Px, Pu, gains = [], [], []
    for j in range(N):
        P = {N: np.asarray(costs.Qx_term[j], float)}
        Kj = {}
        for i in range(N - 1, j, -1):
            Qx, Qu, Qux = costs.Qx[j][i - j - 1], costs.Qu[j][i - j - 1], costs.Qux[j][i - j - 1]
            Bk = Qux + B[i].T @ P[i + 1] @ A[i]
            Kj[i] = -np.linalg.inv(Qu + B[i].T @ P[i + 1] @ B[i]) @ Bk
            P[i] = Qx + A[i].T @ P[i + 1] @ A[i] + Kj[i].T @ Bk
        px = np.zeros((N - j, nx, nx)); pu = np.zeros((max(N - 1 - j, 0), nu, nx))
        gj = np.zeros((max(N - 1 - j, 0), nu, nx))
        px[0] = E[j]
        for i in range(j + 1, N):
            gj[i - j - 1] = Kj[i]
            pu[i - j - 1] = Kj[i] @ px[i - j - 1]
            px[i - j] = (A[i] + B[i] @ Kj[i]) @ px[i - j - 1]
        Px.append(px); Pu.append(pu); gains.append(gj)
    return Response(Px, Pu, gains, N, nx, nu)


# --- robust loops ---------------------------------------------------------------

@dataclass
class RobustSettings:
    sqp: sqp.Settings = field(default_factory=sqp.Settings)
    weights: Weights | None = None
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
    response: Response
    tightening: Tightening
    duals: Duals
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: RobustStats
    qp: lqr.QP


@dataclass
class RobustRtiResult:
    u0: np.ndarray
    warm_start: sqp.Trajectory
    plan: sqp.Trajectory
    tau: Duals
    tightening: Tightening
    response: Response
    lam_stage: np.ndarray
    lam_terminal: np.ndarray
    stats: sqp.Stats


def stage_disturbances(model, traj, inflation=None):
    """sls.py:393-397."""
    E = np.stack([model.disturbance(traj.x[k]) for k in range(traj.N)])
    if inflation is not None:
        E = E + np.stack([inflation(k, traj.x[k]) for k in range(traj.N)])
    return E


def _blend(fresh: Duals, prev: Duals | None, keep: float) -> Duals:
    """sls.py:476-484."""
    if prev is None or keep <= 0.0:
        return fresh
    for j in range(len(fresh.tau)):
        if fresh.tau[j].size:
            fresh.tau[j] = (1 - keep) * fresh.tau[j] + keep * prev.tau[j]
    fresh.tau_term = (1 - keep) * fresh.tau_term + keep * prev.tau_term
    return fresh


def solve_robust(model, x_bar0, s: RobustSettings, initial=None, e_inflation=None):
    """sls.py:400-469."""
    x_bar0 = np.asarray(x_bar0, float)
    w = s.weights or Weights.identity(model.nx, model.nu, s.weight_scale)
    guess, tight, resp, duals = initial, None, None, None
    stats = RobustStats()
    bad_run = 0
    result = None
    last_good = None
    for alt in range(s.max_alternations + 1):
        try:
            nom = sqp.solve_nmpc(model, x_bar0, s.sqp,
                                 guess if guess is not None else sqp.initial_guess(model, x_bar0, 32),
                                 tightenings=tight)
        except sqp.DivergenceError:
            if last_good is None:
                raise
            nom = None
        if nom is None or not nom.stats.converged:
            bad_run += 1
            if bad_run >= 3:
                raise RobustInfeasibleError(
                    "robust problem infeasible: reduce disturbance or relax constraints")
            if nom is None:
                nom = last_good
        else:
            bad_run = 0
            last_good = nom
        stats.sqp_iterations += nom.stats.iterations
        stats.nominal_converged = nom.stats.converged and bad_run == 0
        guess = nom.trajectory
        qp = sqp.linearize(model, nom.trajectory, tight, x_bar0)
        if resp is not None:
            result = RobustResult(nom.trajectory, resp, tight,
                                  duals or Duals.zero(qp.N, qp.nc, qp.nf, s.eps),
                                  nom.lam_stage, nom.lam_terminal, stats, qp)
            if stats.dh <= s.tol_h:
                stats.converged = True
                break
        if alt == s.max_alternations:
            break
        stats.alternations = alt + 1
        if resp is None:
            duals = None
        else:
            fresh = compute_duals(nom.lam_stage, nom.lam_terminal, resp, qp.C, qp.D, qp.CN, s.eps)
            duals = _blend(fresh, duals, s.tau_damping)
        costs = assemble_costs(duals, qp.C, qp.D, qp.CN, w)
        E = stage_disturbances(model, nom.trajectory, e_inflation)
        resp = synthesize(qp.A, qp.B, E, costs)
        nt = tighten(resp, qp.C, qp.D, qp.CN)
        stats.dh = nt.max_abs_diff(tight) if tight is not None and tight.h.shape == nt.h.shape else np.inf
        tight = nt
    return result


def rti_robust_step(model, x_bar0, previous, tau, s: RobustSettings, e_inflation=None,
                    warm_admm=None) -> RobustRtiResult:
    """sls.py:500-525."""
    x_bar0 = np.asarray(x_bar0, float)
    w = s.weights or Weights.identity(model.nx, model.nu, s.weight_scale)
    qp = sqp.linearize(model, previous, None, x_bar0)
    costs = assemble_costs(tau, qp.C, qp.D, qp.CN, w)
    E = stage_disturbances(model, previous, e_inflation)
    resp = synthesize(qp.A, qp.B, E, costs)
    tight = tighten(resp, qp.C, qp.D, qp.CN)
    step = sqp.rti_step(model, x_bar0, previous, s.sqp, tightenings=tight, warm_admm=warm_admm)
    tau_next = compute_duals(step.lam_stage, step.lam_terminal, resp, qp.C, qp.D, qp.CN, s.eps)
    return RobustRtiResult(step.u0, step.warm_start, step.plan, tau_next, tight, resp,
                           step.lam_stage, step.lam_terminal, step.stats)
