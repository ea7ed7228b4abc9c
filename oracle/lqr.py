"""Oracle (test infrastructure): LTV-LQR by conditional-value-function scans.

Restates /root/reference/pkg/src/scanmpc/lqr.py in float64 numpy:

* QP container and validation ............ lqr.py:43-113
* SPD inverse with pivot/ridge rule ...... lqr.py:185-220
* CVF combine (Eq. 28) ................... lqr.py:226-262
* COT combine ............................ lqr.py:273-291
* leaves (Eq. 29), gains, assembly ....... lqr.py:297-363
* full solve / cache build / replay ...... lqr.py:366-454
* relative error metric .................. reference.py:23-29
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import tree

RCOND_MIN = 1e-14
PIVOT_MIN = 1e-10
RIDGE = 1e-9


class IllConditionedCombineError(ArithmeticError):
    pass


class SingularStageError(ArithmeticError):
    pass


class CacheInvalidatedError(RuntimeError):
    pass


def relative_error(actual, expected) -> float:
    """max|a - e| / max(1, max|e|)  (reference.py:23-29)."""
    actual = np.asarray(actual, float)
    expected = np.asarray(expected, float)
    if actual.size == 0:
        return 0.0
    scale = max(1.0, float(np.abs(expected).max())) if expected.size else 1.0
    return float(np.abs(actual - expected).max() / scale)


@dataclass
class QP:
    """Stagewise LTV-QP data, same field names/shapes as lqr.py:53-68."""

    A: np.ndarray
    B: np.ndarray
    b: np.ndarray
    Q: np.ndarray
    R: np.ndarray
    S: np.ndarray
    q: np.ndarray
    r: np.ndarray
    QN: np.ndarray
    qN: np.ndarray
    C: np.ndarray
    D: np.ndarray
    f: np.ndarray
    CN: np.ndarray
    fN: np.ndarray
    dx0: np.ndarray

    @property
    def N(self):
        return self.A.shape[0]

    @property
    def nx(self):
        return self.QN.shape[0]

    @property
    def nu(self):
        return self.R.shape[-1] if self.N > 0 else self.S.shape[1]

    @property
    def nc(self):
        return self.C.shape[1]

    @property
    def nf(self):
        return self.CN.shape[0]

    def replace(self, **kw) -> "QP":
        d = dict(self.__dict__)
        d.update(kw)
        return QP(**d)

    @classmethod
    def of(cls, other) -> "QP":
        return cls(**{k: np.asarray(getattr(other, k), float) for k in FIELDS})


FIELDS = ("A", "B", "b", "Q", "R", "S", "q", "r", "QN", "qN", "C", "D", "f", "CN", "fN", "dx0")


@dataclass
class Solution:
    dx: np.ndarray
    du: np.ndarray
    K: np.ndarray
    k: np.ndarray
    P: np.ndarray
    p: np.ndarray
    scan_layers: int = 0


@dataclass
class Cache:
    generation: int
    stat: dict
    K: np.ndarray
    Gamma: np.ndarray
    P: np.ndarray
    Abar: np.ndarray
    cvf_tape: list = field(default_factory=list)
    cot_tape: list = field(default_factory=list)
    scan_layers: int = 0


def _mv(M, v):
    return (M @ v[..., None])[..., 0]


def _T(M):
    return np.ascontiguousarray(np.swapaxes(M, -1, -2))


def spd_inverse(M, label="matrix"):
    """Cholesky-based inverse; pivot^2 < 1e-10 -> ridge 1e-9 -> error (lqr.py:185-220)."""
    M = np.asarray(M, dtype=float)
    k = M.shape[-1]
    stack = M.reshape((-1, k, k))
    need_loop = False
    try:
        L = np.linalg.cholesky(stack)
        piv2 = np.diagonal(L, axis1=-2, axis2=-1) ** 2
        need_loop = bool((piv2.min(axis=-1) < PIVOT_MIN).any()) if stack.shape[0] else False
    except np.linalg.LinAlgError:
        need_loop = True
    if need_loop:
        L = np.empty_like(stack)
        for i in range(stack.shape[0]):
            try:
                Li = np.linalg.cholesky(stack[i])
                if (np.diag(Li) ** 2).min() < PIVOT_MIN:
                    raise np.linalg.LinAlgError
            except np.linalg.LinAlgError:
                try:
                    Li = np.linalg.cholesky(stack[i] + RIDGE * np.eye(k))
                except np.linalg.LinAlgError as exc:
                    raise SingularStageError(f"singular {label} at stage {i}") from exc
            L[i] = Li
    eye = np.broadcast_to(np.eye(k), stack.shape)
    Linv = np.linalg.solve(L, np.ascontiguousarray(eye))
    return (_T(Linv) @ Linv).reshape(M.shape)


# --- CVF / COT combines ------------------------------------------------------

def cvf_matrix(Pl, Al, Cl, Pr, Ar, Cr):
    """Matrix half of Eq. 28 (lqr.py:226-239)."""
    eye = np.broadcast_to(np.eye(Pl.shape[-1]), Pl.shape)
    M1 = eye + Pr @ Cl
    if not np.all(1.0 / np.linalg.cond(M1) > RCOND_MIN):
        raise IllConditionedCombineError("ill-conditioned combine")
    M2 = eye + Cl @ Pr
    Ups = _T(np.linalg.solve(_T(M1), Al))
    Psi = _T(np.linalg.solve(_T(M2), _T(Ar)))
    P = Ups @ Pr @ Al + Pl
    A = Psi @ Al
    C = Psi @ Cl @ _T(Ar) + Cr
    return P, A, C, Ups, Psi


def cvf_affine(Ups, Pr, Psi, Cl, pl, bl, pr, br):
    """Vector half of Eq. 28 (lqr.py:242-246)."""
    p = _mv(Ups, pr + _mv(Pr, bl)) + pl
    b = _mv(Psi, bl - _mv(Cl, pr)) + br
    return p, b


def cvf_op(lhs, rhs):
    Pl, pl, Al, Cl, bl = lhs
    Pr, pr, Ar, Cr, br = rhs
    P, A, C, Ups, Psi = cvf_matrix(Pl, Al, Cl, Pr, Ar, Cr)
    p, b = cvf_affine(Ups, Pr, Psi, Cl, pl, bl, pr, br)
    return (P, p, A, C, b), (Ups, Pr, Psi, Cl)


def cvf_replay_op(lhs, rhs, aux):
    Ups, Pr, Psi, Cl = aux
    return cvf_affine(Ups, Pr, Psi, Cl, lhs[0], lhs[1], rhs[0], rhs[1]), ()


def cvf_unit(k, n, grid=()):
    shp = (k,) + tuple(grid)
    I = np.zeros(shp + (n, n))
    I[...] = np.eye(n)
    return (np.zeros(shp + (n, n)), np.zeros(shp + (n,)), I, np.zeros(shp + (n, n)), np.zeros(shp + (n,)))


def cot_op(lhs, rhs):
    return (rhs[0] @ lhs[0], _mv(rhs[0], lhs[1]) + rhs[1]), (rhs[0],)


def cot_replay_op(lhs, rhs, aux):
    return (_mv(aux[0], lhs[0]) + rhs[0],), ()


def cot_unit(k, n):
    I = np.zeros((k, n, n))
    I[...] = np.eye(n)
    return (I, np.zeros((k, n)))


# --- leaves, gains, assembly --------------------------------------------------

def static_terms(qp: QP) -> dict:
    """Penalty-invariant stage terms (lqr.py:314-335)."""
    N, n, m = qp.N, qp.nx, qp.nu
    if N == 0:
        z = np.zeros((0, n, n))
        return dict(A=qp.A, B=qp.B, BT=np.zeros((0, m, n)), b=qp.b, dx0=np.asarray(qp.dx0, float),
                    Rinv=np.zeros((0, m, m)), ST=np.zeros((0, n, m)), P0=z, A0=z, C0=z,
                    QN=np.asarray(qp.QN, float))
    Rinv = spd_inverse(qp.R, "R")
    ST = _T(qp.S)
    BT = _T(qp.B)
    RS = Rinv @ qp.S
    return dict(A=np.ascontiguousarray(qp.A), B=np.ascontiguousarray(qp.B), BT=BT,
                b=np.ascontiguousarray(qp.b), dx0=np.asarray(qp.dx0, float), Rinv=Rinv, ST=ST,
                P0=np.ascontiguousarray(qp.Q - ST @ RS),
                A0=np.ascontiguousarray(qp.A - qp.B @ RS),
                C0=np.ascontiguousarray(qp.B @ Rinv @ BT), QN=np.asarray(qp.QN, float))


def leaf_vectors(st, q, r):
    """lqr.py:338-342."""
    w = _mv(st["Rinv"], np.asarray(r, float))
    return np.asarray(q, float) - _mv(st["ST"], w), st["b"] - _mv(st["B"], w)


def leaves(qp: QP):
    """Eq. 29 scan elements, stages then terminal (lqr.py:297-311)."""
    st = static_terms(qp)
    p0, b0 = leaf_vectors(st, qp.q, qp.r)
    n = qp.nx
    zm = np.zeros((1, n, n))
    elems = (np.concatenate([st["P0"], st["QN"][None]]),
             np.concatenate([p0, np.asarray(qp.qN, float)[None]]),
             np.concatenate([st["A0"], zm]),
             np.concatenate([st["C0"], zm]),
             np.concatenate([b0, np.zeros((1, n))]))
    return elems, st


def feedforward(Gamma, BT, Pn, b, pn, r):
    """lqr.py:345-346."""
    return -_mv(Gamma, _mv(BT, pn + _mv(Pn, b)) + np.asarray(r, float))


def cot_leaves(st, Abar, k):
    """lqr.py:349-356."""
    bb = _mv(st["B"], k) + st["b"]
    Ael = Abar.copy()
    bel = bb.copy()
    Ael[0] = 0.0
    bel[0] = Abar[0] @ st["dx0"] + bb[0]
    return np.ascontiguousarray(Ael), np.ascontiguousarray(bel)


def _finish(st, K, k, xs, p, P, tally):
    N = K.shape[0]
    dx = np.concatenate([st["dx0"][None], xs]) if N else st["dx0"][None]
    du = _mv(K, dx[:-1]) + k if N else np.zeros((0, 0))
    return Solution(dx=dx, du=du, K=K, k=k, P=P, p=p, scan_layers=tally.layers)


def _solve(qp: QP, record: bool):
    N, n, m = qp.N, qp.nx, qp.nu
    elems, st = leaves(qp)
    tally = tree.Tally()
    out, tape = tree.scan(elems, cvf_op, lambda c: cvf_unit(c, n), reverse=True,
                          record=record, tally=tally)
    P, p = out[0], out[1]
    if N == 0:
        sol = Solution(dx=st["dx0"][None], du=np.zeros((0, m)), K=np.zeros((0, m, n)),
                       k=np.zeros((0, m)), P=P, p=p, scan_layers=tally.layers)
        cache = Cache(0, st, sol.K, np.zeros((0, m, m)), P, np.zeros((0, n, n)), [], [],
                      tally.layers) if record else None
        return sol, cache
    Pn, pn = np.ascontiguousarray(P[1:]), np.ascontiguousarray(p[1:])
    Gamma = spd_inverse(qp.R + st["BT"] @ Pn @ st["B"], "R + B'PB")
    K = np.ascontiguousarray(-(Gamma @ (qp.S + st["BT"] @ Pn @ st["A"])))
    k = feedforward(Gamma, st["BT"], Pn, st["b"], pn, qp.r)
    Abar = np.ascontiguousarray(st["A"] + st["B"] @ K)
    cot_out, cot_tape = tree.scan(cot_leaves(st, Abar, k), cot_op, lambda c: cot_unit(c, n),
                                  record=record)
    sol = _finish(st, K, k, cot_out[1], p, P, tally)
    cache = Cache(0, st, K, Gamma, P, Abar, tape, cot_tape, tally.layers) if record else None
    return sol, cache


def solve(qp) -> Solution:
    """lqr.py:366-369."""
    return _solve(QP.of(qp), False)[0]


def build_cache(qp, generation: int = 0):
    """lqr.py:372-376."""
    sol, cache = _solve(QP.of(qp), True)
    cache.generation = generation
    return sol, cache


def solve_cached(q, r, qN, cache: Cache, generation: int) -> Solution:
    """Replay with new linear terms only (lqr.py:419-454)."""
    if generation != cache.generation:
        raise CacheInvalidatedError("cache invalidated")
    st = cache.stat
    N, n = st["A"].shape[0], st["QN"].shape[0]
    p0, b0 = leaf_vectors(st, q, r)
    pel = np.concatenate([p0, np.asarray(qN, float)[None]])
    bel = np.concatenate([b0, np.zeros((1, n))])
    tally = tree.Tally()
    out, _ = tree.scan((pel, bel), cvf_replay_op, lambda c: (np.zeros((c, n)), np.zeros((c, n))),
                       reverse=True, replay=cache.cvf_tape, tally=tally)
    p = out[0]
    if N == 0:
        return Solution(dx=st["dx0"][None], du=np.zeros((0, 0)), K=cache.K, k=np.zeros((0, 0)),
                        P=cache.P, p=p, scan_layers=tally.layers)
    k = feedforward(cache.Gamma, st["BT"], np.ascontiguousarray(cache.P[1:]), st["b"],
                    np.ascontiguousarray(p[1:]), r)
    _, bcot = cot_leaves(st, cache.Abar, k)
    cot_out, _ = tree.scan((bcot,), cot_replay_op, lambda c: (np.zeros((c, n)),),
                           replay=cache.cot_tape)
    return _finish(st, cache.K, k, cot_out[0], p, cache.P, tally)


def riccati(qp) -> Solution:
    """Sequential textbook Riccati recursion (reference.py:32-62), independent check."""
    qp = QP.of(qp)
    N, n, m = qp.N, qp.nx, qp.nu
    P = np.zeros((N + 1, n, n)); p = np.zeros((N + 1, n))
    K = np.zeros((N, m, n)); k = np.zeros((N, m))
    P[N], p[N] = qp.QN, qp.qN
    for i in range(N - 1, -1, -1):
        A, B, b = qp.A[i], qp.B[i], qp.b[i]
        H = qp.R[i] + B.T @ P[i + 1] @ B
        G = qp.S[i] + B.T @ P[i + 1] @ A
        K[i] = -np.linalg.solve(H, G)
        k[i] = -np.linalg.solve(H, B.T @ (p[i + 1] + P[i + 1] @ b) + qp.r[i])
        P[i] = qp.Q[i] + A.T @ P[i + 1] @ A + G.T @ K[i]
        p[i] = qp.q[i] + A.T @ (p[i + 1] + P[i + 1] @ b) + G.T @ k[i]
    dx = np.zeros((N + 1, n)); du = np.zeros((N, m))
    dx[0] = qp.dx0
    for i in range(N):
        du[i] = K[i] @ dx[i] + k[i]
        dx[i + 1] = qp.A[i] @ dx[i] + qp.B[i] @ du[i] + qp.b[i]
    return Solution(dx=dx, du=du, K=K, k=k, P=P, p=p)
