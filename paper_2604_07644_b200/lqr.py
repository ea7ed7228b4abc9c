"""Drop-in for ``scanmpc.lqr``: LTV-LQR by CVF / COT associative scans on the GPU.

Same names, signatures and dataclasses as /root/reference/pkg/src/scanmpc/lqr.py:
``LtvQpData`` (lqr.py:43-113), ``LqrLinearTerms`` (:116), ``LqrSolution`` (:123),
``LqrCache`` (:157), ``solve`` (:366), ``build_cache`` (:372),
``solve_cached`` (:419) and the error classes (:31-40).

The factorization (CVF leaves, the reverse combine tree with recorded
Ups/Pr/Psi/Cl, gains, the forward COT tree) runs in csrc/lqr.cu; every vector
quantity comes from the replay kernel in csrc/admm.cu, so ``solve`` and
``solve_cached`` produce bitwise-identical results for the same linear terms.
numpy inputs give float64 numpy outputs (computed in float32 on the device);
CUDA tensor inputs give tensors.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .device import Context, DeviceQp, resolve, stream_ptr, to_dev, to_host
from .errors import CacheInvalidatedError, IllConditionedCombineError, SingularStageError  # noqa: F401
from .scan import scan_depth

RCOND_COMBINE = 1e-14
CHOL_PIVOT_MIN = 1e-10
CHOL_REG = 1e-9


@dataclass
class LtvQpData:
    """Stagewise QP data (lqr.py:43-68); arrays may be numpy or torch."""

    A: object
    B: object
    b: object
    Q: object
    R: object
    S: object
    q: object
    r: object
    QN: object
    qN: object
    C: object
    D: object
    f: object
    CN: object
    fN: object
    dx0: object

    @property
    def N(self) -> int:
        return self.A.shape[0]

    @property
    def nx(self) -> int:
        return self.QN.shape[0]

    @property
    def nu(self) -> int:
        return self.R.shape[-1] if self.N > 0 else self.S.shape[1]

    @property
    def nc(self) -> int:
        return self.C.shape[1]

    @property
    def nf(self) -> int:
        return self.CN.shape[0]

    def validate(self) -> None:
        """lqr.py:90-106."""
        N, nx, nu, nc, nf = self.N, self.nx, self.nu, self.nc, self.nf
        expect = {"A": (N, nx, nx), "B": (N, nx, nu), "b": (N, nx), "Q": (N, nx, nx), "R": (N, nu, nu),
                  "S": (N, nu, nx), "q": (N, nx), "r": (N, nu), "QN": (nx, nx), "qN": (nx,),
                  "C": (N, nc, nx), "D": (N, nc, nu), "f": (N, nc), "CN": (nf, nx), "fN": (nf,),
                  "dx0": (nx,)}
        for name, shape in expect.items():
            got = tuple(getattr(self, name).shape)
            if got != shape:
                raise ValueError(f"{name} has shape {got}, expected {shape}")
        Q = np.asarray(self.Q.cpu() if isinstance(self.Q, torch.Tensor) else self.Q)
        QN = np.asarray(self.QN.cpu() if isinstance(self.QN, torch.Tensor) else self.QN)
        if N > 0 and not np.allclose(Q, np.swapaxes(Q, -1, -2)):
            raise ValueError("Q stages must be symmetric")
        if not np.allclose(QN, QN.T):
            raise ValueError("QN must be symmetric")

    def with_linear_terms(self, q, r, qN) -> "LtvQpData":
        return LtvQpData(A=self.A, B=self.B, b=self.b, Q=self.Q, R=self.R, S=self.S, q=q, r=r, QN=self.QN,
                         qN=qN, C=self.C, D=self.D, f=self.f, CN=self.CN, fN=self.fN, dx0=self.dx0)


@dataclass
class LqrLinearTerms:
    q: object
    r: object
    qN: object


@dataclass
class LqrSolution:
    dx: object
    du: object
    K: object
    k: object
    P: object
    p: object
    scan_layers: int = 0

    def dynamics_residual(self, qp) -> float:
        """lqr.py:133-137."""
        if qp.N == 0:
            return 0.0
        A, B, b = (np.asarray(getattr(qp, k)) for k in ("A", "B", "b"))
        dx, du = np.asarray(self.dx), np.asarray(self.du)
        pred = (A @ dx[:-1, :, None])[..., 0] + (B @ du[..., None])[..., 0] + b
        return float(np.abs(dx[1:] - pred).max())


class LqrCache:
    """Device-resident factorization (lqr.py:157-169), stamped by generation.

    Owns its own solver context, so later solves do not disturb it; the
    static data (A, B, b, S, dx0) of the QP it was built from stay bound.
    """

    def __init__(self, ctx: Context, dqp: DeviceQp, generation: int, scan_layers: int, as_numpy: bool):
        self.ctx = ctx
        self.dqp = dqp
        self.generation = generation
        self.scan_layers = scan_layers
        self._numpy = as_numpy


def _is_torch(qp) -> bool:
    return isinstance(qp.QN, torch.Tensor)


def _outputs(N, n, m, batch=1, full=True):
    dev = torch.device("cuda", torch.cuda.current_device())
    d = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
    z = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
    out = {"dx": d(batch, N + 1, n), "du": d(batch, N, m), "k": d(batch, N, m), "p": d(batch, N + 1, n)}
    if full:
        out["K"] = z(batch, N, m, n)
        out["P"] = z(batch, N + 1, n, n)
    return out


def _finish(out: dict, K, P, layers: int, as_numpy: bool) -> LqrSolution:
    conv = (lambda t: to_host(t[0])) if as_numpy else (lambda t: t[0])
    return LqrSolution(dx=conv(out["dx"]), du=conv(out["du"]), K=conv(K), k=conv(out["k"]), P=conv(P),
                       p=conv(out["p"]), scan_layers=layers)


def _dims(qp):
    return qp.nx, qp.nu, qp.nc, qp.nf, qp.N


def _solve(qp, executor, generation, own_ctx: bool):
    dev = resolve(executor)
    n, m, c, nf, N = _dims(qp)
    ctx = Context(n, m, c, nf, N, 1) if own_ctx else dev.context(n, m, c, nf, N, 1)
    dqp = DeviceQp.from_host(qp)
    out = _outputs(N, n, m)
    s = dqp.cstruct()
    rc = ctx.lib.gsls_lqr_solve(ctx.handle, ctypes.byref(s), int(generation), out["dx"].data_ptr(),
                                out["du"].data_ptr() if N else None, out["K"].data_ptr() if N else None,
                                out["k"].data_ptr() if N else None, out["P"].data_ptr(), out["p"].data_ptr(),
                                stream_ptr())
    nat.check(rc, "lqr.solve")
    sol = _finish(out, out["K"], out["P"], scan_depth(N + 1), not _is_torch(qp))
    return sol, ctx, dqp


def solve(qp, executor=None) -> LqrSolution:
    """Solve the equality-constrained LTV-QP by reverse CVF / forward COT scans (lqr.py:366)."""
    return _solve(qp, executor, 0, own_ctx=False)[0]


def build_cache(qp, executor=None, generation: int = 0):
    """Full solve that also keeps every penalty-invariant intermediate (lqr.py:372)."""
    sol, ctx, dqp = _solve(qp, executor, generation, own_ctx=True)
    cache = LqrCache(ctx, dqp, generation, sol.scan_layers, not _is_torch(qp))
    cache.K, cache.P = sol.K, sol.P
    return sol, cache


def solve_cached(lin: LqrLinearTerms, cache: LqrCache, generation: int, executor=None) -> LqrSolution:
    """Replay the recorded scans with new linear terms only (lqr.py:419).

    Raises CacheInvalidatedError("cache invalidated") on a generation mismatch.
    """
    if generation != cache.generation:
        raise CacheInvalidatedError("cache invalidated")
    ctx, dqp = cache.ctx, cache.dqp
    d = ctx.dims
    q = to_dev(lin.q, torch.float64).reshape(1, d.N, d.nx)
    r = to_dev(lin.r, torch.float64).reshape(1, d.N, d.nu)
    qN = to_dev(lin.qN, torch.float64).reshape(1, d.nx)
    out = _outputs(d.N, d.nx, d.nu, full=False)
    s = dqp.cstruct()
    rc = ctx.lib.gsls_lqr_solve_cached(ctx.handle, ctypes.byref(s), q.data_ptr() if q.numel() else None,
                                       r.data_ptr() if r.numel() else None, qN.data_ptr(), int(generation),
                                       out["dx"].data_ptr(), out["du"].data_ptr() if d.N else None,
                                       out["k"].data_ptr() if d.N else None, out["p"].data_ptr(), stream_ptr())
    nat.check(rc, "lqr.solve_cached")
    conv = (lambda t: to_host(t[0])) if cache._numpy else (lambda t: t[0])
    return LqrSolution(dx=conv(out["dx"]), du=conv(out["du"]), K=cache.K, k=conv(out["k"]), P=cache.P,
                       p=conv(out["p"]), scan_layers=cache.scan_layers)
