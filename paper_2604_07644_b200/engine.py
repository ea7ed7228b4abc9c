"""Batched, device-resident MPC steps: the hot path of the metric.

``RtiEngine`` runs B independent instances of one plant through
``sls.rti_robust_step`` (sls.py:500-525) — or the nominal ``sqp.rti_step``
(sqp.py:272-302) when ``robust=False`` — entirely on one GPU:

    linearize (csrc/models.cu)
    -> assemble_costs -> synthesize -> tighten (csrc/sls.cu)
    -> f -= h (tightened re-linearization)
    -> ADMM QP with cached factorizations (csrc/lqr.cu, csrc/admm.cu)
    -> compute_duals (tau for the next step) -> plan / warm start / u0

Every buffer is allocated once per engine; a step issues only kernel
launches plus the ADMM driver's per-rebuild status read.  The drop-in
functions in ``sls`` / ``sqp`` wrap an engine with batch 1.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .admm import AdmmSettings, DeviceAdmmState, DeviceAdmmStats
from .device import Context, DeviceQp, field_dtype, stream_ptr, to_dev

F32, F64 = torch.float32, torch.float64


def _p(t):
    return t.data_ptr() if (t is not None and t.numel()) else None


class DeviceModel:
    """Device twin of a plant: parameters, weights and reference uploaded once."""

    def __init__(self, model, N: int):
        spec = model.device_spec()
        if spec is None:
            raise TypeError(f"{type(model).__name__} has no device twin (device_spec() is None)")
        mid, mparams, cparams = spec
        self.model = model
        self.model_id = int(mid)
        self.params = to_dev(np.concatenate([np.asarray(mparams, float), np.asarray(cparams, float)]), F64)
        self.cons_offset = len(mparams)
        self.nx, self.nu, self.nc, self.nf, self.N = model.nx, model.nu, model.nc, model.nf, N
        Q, R, QN = model.cost_weights()
        xref, uref = model.reference(N)
        self.Qw, self.Rw, self.QNw = (to_dev(np.asarray(a, float), F64) for a in (Q, R, QN))
        self.xref, self.uref = to_dev(xref, F64), to_dev(uref, F64)
        self.E = to_dev(np.asarray(model.disturbance(np.zeros(self.nx)), float), F64)


def alloc_qp(B, n, m, c, nf, N, device=None) -> DeviceQp:
    dev = device or torch.device("cuda", torch.cuda.current_device())
    shapes = {"A": (B, N, n, n), "B": (B, N, n, m), "b": (B, N, n), "Q": (B, N, n, n), "R": (B, N, m, m),
              "S": (B, N, m, n), "q": (B, N, n), "r": (B, N, m), "QN": (B, n, n), "qN": (B, n),
              "C": (B, N, c, n), "D": (B, N, c, m), "f": (B, N, c), "CN": (B, nf, n), "fN": (B, nf),
              "dx0": (B, n)}
    return DeviceQp(**{k: torch.zeros(s, dtype=field_dtype(k), device=dev) for k, s in shapes.items()})


def linearize_into(ctx: Context, dm: DeviceModel, qp: DeviceQp, x, u, h=None, hf=None, xbar0=None, E=None,
                   write_weights: bool = True):
    """sqp.linearize (sqp.py:105-147) of a batch of trajectories into ``qp`` (device)."""
    a = nat.LinArgs()
    a.model_id = dm.model_id
    a.params = dm.params.data_ptr()
    a.cons_offset = dm.cons_offset
    a.x, a.u = x.data_ptr(), u.data_ptr()
    a.h, a.hf = _p(h), _p(hf)
    a.xbar0 = _p(xbar0)
    a.Qw, a.Rw, a.QNw = dm.Qw.data_ptr(), dm.Rw.data_ptr(), dm.QNw.data_ptr()
    a.xref, a.uref = dm.xref.data_ptr(), dm.uref.data_ptr()
    a.E_const = dm.E.data_ptr()
    a.write_weights = int(write_weights)
    s = qp.cstruct()
    nat.check(ctx.lib.gsls_linearize(ctx.handle, ctypes.byref(a), ctypes.byref(s), _p(E), stream_ptr()),
              "linearize")


class RtiEngine:
    """B instances of one plant, one robust (or nominal) RTI step per call."""

    def __init__(self, model, N: int, batch: int, settings, robust: bool = True):
        """``settings`` is an ``sls.RobustSettings`` (robust) or ``sqp.SqpSettings`` (nominal)."""
        nat.load()
        self.model = model
        self.robust = robust
        self.settings = settings
        sqp_set = settings.sqp if robust else settings
        self.admm_settings: AdmmSettings = sqp_set.admm
        n, m, c, nf = model.nx, model.nu, model.nc, model.nf
        self.dims = (n, m, c, nf, N)
        self.B = batch
        self.ctx = Context(n, m, c, nf, N, batch)
        self.dm = DeviceModel(model, N)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.qp = alloc_qp(batch, n, m, c, nf, N, dev)
        self.mtot = N * c + nf
        self.ncell = N * (N + 1) // 2
        self.E = torch.zeros(batch, N, n, n, dtype=F32, device=dev)
        self.h = torch.zeros(batch, N, c, dtype=F64, device=dev)
        self.hf = torch.zeros(batch, nf, dtype=F64, device=dev)
        self.tau = torch.zeros(batch, self.ncell, c, dtype=F64, device=dev)
        self.tau_term = torch.zeros(batch, N, nf, dtype=F64, device=dev)
        self.beta = torch.zeros_like(self.tau)
        self.beta_term = torch.zeros_like(self.tau_term)
        self.tau_valid = False
        if robust:
            w = settings.weights
            if w is None:
                s = settings.weight_scale
                Qb, Rb, QbN = s * np.eye(n), s * np.eye(m), s * np.eye(n)
            else:
                Qb, Rb, QbN = w.Qbar, w.Rbar, w.QbarN
            self.Qbar, self.Rbar, self.QbarN = (to_dev(np.asarray(a, float), F32) for a in (Qb, Rb, QbN))
        self.state = DeviceAdmmState(batch, self.mtot, self.admm_settings.rho0, dev)
        self.stats = DeviceAdmmStats(batch, dev)
        d = lambda *s: torch.zeros(s, dtype=F64, device=dev)  # noqa: E731
        self.dx, self.du = d(batch, N + 1, n), d(batch, N, m)
        self.plan_x, self.plan_u = d(batch, N + 1, n), d(batch, N, m)
        self.warm_x, self.warm_u = d(batch, N + 1, n), d(batch, N, m)
        self.u0 = d(batch, m)
        self.cost = d(batch)
        self._weights_written = False
        self.launches_per_step = 0
        # the ADMM's first cache build runs on the context's side stream, overlapped with the
        # SLS synthesis (csrc/rti.cu); GSLS_OVERLAP=0 serializes it (phase timing)
        import os
        self.overlap = robust and os.environ.get("GSLS_OVERLAP", "1") != "0"

    def step(self, xbar0: torch.Tensor, prev_x: torch.Tensor, prev_u: torch.Tensor, tau=None, tau_term=None,
             use_tau: bool | None = None, E: torch.Tensor | None = None, warm_admm: bool = False):
        """One step for every instance.  Inputs are float64 CUDA tensors
        (B,n), (B,N+1,n), (B,N,m); ``tau``/``tau_term`` (cell layout) override the
        engine-held duals; ``use_tau=False`` forces the unweighted synthesis."""
        ctx, lib, qp, S = self.ctx, self.ctx.lib, self.qp, stream_ptr()
        n, m, c, nf, N = self.dims
        for name, t, shape in (("xbar0", xbar0, (self.B, n)), ("prev_x", prev_x, (self.B, N + 1, n)),
                               ("prev_u", prev_u, (self.B, N, m)), ("tau", tau, (self.B, self.ncell, c)),
                               ("tau_term", tau_term, (self.B, N, nf))):
            if t is not None and (tuple(t.shape) != shape or t.dtype != F64 or not t.is_cuda or not t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous float64 CUDA tensor of shape {shape}, "
                                 f"got {tuple(t.shape)} {t.dtype} contiguous={t.is_contiguous()}")
        # the whole step is one C-ABI call (csrc/rti.cu): linearize -> [SLS chain, with the
        # ADMM's first factorization on the context's side stream] -> ADMM -> duals -> plan
        a = nat.RtiStepArgs()
        dm = self.dm
        a.lin.model_id, a.lin.params, a.lin.cons_offset = dm.model_id, dm.params.data_ptr(), dm.cons_offset
        a.lin.x, a.lin.u, a.lin.h, a.lin.hf, a.lin.xbar0 = prev_x.data_ptr(), prev_u.data_ptr(), None, None, _p(xbar0)
        a.lin.Qw, a.lin.Rw, a.lin.QNw = dm.Qw.data_ptr(), dm.Rw.data_ptr(), dm.QNw.data_ptr()
        a.lin.xref, a.lin.uref, a.lin.E_const = dm.xref.data_ptr(), dm.uref.data_ptr(), dm.E.data_ptr()
        a.lin.write_weights = int(not self._weights_written)
        qs = qp.cstruct()
        a.qp = ctypes.pointer(qs)
        a.E, a.E_in = self.E.data_ptr(), _p(E)
        a.robust, a.warm_admm, a.no_overlap = int(self.robust), int(warm_admm), int(not self.overlap)
        if self.robust:
            if tau is not None:
                self.tau.copy_(tau)
                self.tau_term.copy_(tau_term)
                self.tau_valid = True
            if use_tau is None:
                use_tau = self.tau_valid
            a.use_tau = int(bool(use_tau))
            a.Qbar, a.Rbar, a.QbarN = self.Qbar.data_ptr(), self.Rbar.data_ptr(), self.QbarN.data_ptr()
            a.tau, a.tau_term, a.beta, a.beta_term = (_p(t) for t in (self.tau, self.tau_term, self.beta,
                                                                      self.beta_term))
            a.eps = float(self.settings.eps)
            a.h, a.hf = _p(self.h), _p(self.hf)
        a.admm, a.state, a.stats = self.admm_settings.cstruct(), self.state.cstruct(), self.stats.cstruct()
        a.dx, a.du = self.dx.data_ptr(), _p(self.du)
        a.plan_x, a.plan_u, a.warm_x, a.warm_u = (t.data_ptr() for t in (self.plan_x, self.plan_u, self.warm_x,
                                                                          self.warm_u))
        a.u0, a.cost = self.u0.data_ptr(), self.cost.data_ptr()
        nat.check(lib.gsls_rti_step(ctx.handle, ctypes.byref(a), S), "rti step")
        self._weights_written = True
        if self.robust:
            self.tau_valid = True
        return self

    def capture(self, xbar0=None, prev_x=None, prev_u=None) -> "CapturedStep":
        """Record one step of this engine as a CUDA graph (see CapturedStep)."""
        return CapturedStep(self, xbar0, prev_x, prev_u)

    # -- views ---------------------------------------------------------------------
    def lam_split(self):
        n, m, c, nf, N = self.dims
        return self.state.lam[:, : N * c].reshape(self.B, N, c), self.state.lam[:, N * c:]

    def export_response(self):
        """(phix (B,ncell,n,n), phiu, gains (B,ncell,m,n)) float32 device tensors."""
        n, m, c, nf, N = self.dims
        dev = self.qp.QN.device
        phix = torch.empty(self.B, self.ncell, n, n, dtype=F32, device=dev)
        phiu = torch.empty(self.B, self.ncell, m, n, dtype=F32, device=dev)
        gains = torch.empty_like(phiu)
        nat.check(self.ctx.lib.gsls_sls_export(self.ctx.handle, phix.data_ptr(), phiu.data_ptr(),
                                               gains.data_ptr(), stream_ptr()), "sls export")
        return phix, phiu, gains


class CapturedStep:
    """One MPC step of an ``RtiEngine`` recorded as a single CUDA graph.

    The graph holds the whole step: linearization, the SLS chain (and the ADMM's first
    factorization on a forked branch), the ADMM QP as a conditional WHILE node over
    [rebuild | persistent replay | decide] (csrc/admm.cu admm_solve_captured), duals and
    the plan update.  A replay issues one graph launch and no host synchronization;
    ``check()`` reads the error records afterwards (one D2H copy), raising as the eager
    step would.  Inputs are copied into static device buffers; the engine-held duals
    carry over between steps as in the eager receding-horizon loop.

    A step whose factored SLS combine met an indefinite P (GSLS_ERR_LOWRANK) switched the
    context to dense combines: the recorded graph is then stale, so ``check()`` re-runs the
    step eagerly and re-records the graph.
    """

    def __init__(self, eng: RtiEngine, xbar0=None, prev_x=None, prev_u=None):
        n, m, c, nf, N = eng.dims
        dev = eng.qp.QN.device
        self.eng = eng
        z = lambda *s: torch.zeros(s, dtype=F64, device=dev)  # noqa: E731
        self.xbar0, self.prev_x, self.prev_u = z(eng.B, n), z(eng.B, N + 1, n), z(eng.B, N, m)
        if xbar0 is not None:
            self._load(xbar0, prev_x, prev_u)
        self._record()

    def _load(self, xbar0, prev_x, prev_u):
        self.xbar0.copy_(xbar0, non_blocking=True)
        self.prev_x.copy_(prev_x, non_blocking=True)
        self.prev_u.copy_(prev_u, non_blocking=True)

    def _record(self):
        eng = self.eng
        if eng.robust and not eng.tau_valid:
            raise RuntimeError("capture after one eager robust step (the duals tau must be valid)")
        s = torch.cuda.Stream(device=self.xbar0.device)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up on the capture stream: lazy allocations / attributes
            eng.step(self.xbar0, self.prev_x, self.prev_u)
        s.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=s, capture_error_mode="relaxed"):
            eng.step(self.xbar0, self.prev_x, self.prev_u)
        torch.cuda.current_stream().wait_stream(s)

    def __call__(self, xbar0=None, prev_x=None, prev_u=None) -> RtiEngine:
        if xbar0 is not None:
            self._load(xbar0, prev_x, prev_u)
        self.graph.replay()
        return self.eng

    def check(self):
        """Raise the step's error, if any (synchronizes)."""
        eng = self.eng
        rc = eng.ctx.lib.gsls_ctx_check(eng.ctx.handle, stream_ptr())
        if rc == nat.ERR_LOWRANK:  # the context now runs dense combines: re-run eagerly, re-record
            eng.step(self.xbar0, self.prev_x, self.prev_u)
            nat.check(eng.ctx.lib.gsls_ctx_check(eng.ctx.handle, stream_ptr()), "graph step")
            self._record()
            return
        nat.check(rc, "graph step")
