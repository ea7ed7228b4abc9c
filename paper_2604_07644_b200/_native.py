"""ctypes binding of libgsls.so (the C ABI in include/gsls.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
CPU fallback: importing the product path without the library, or without a
CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSLS_LIB") or os.path.join(_HERE, "libgsls.so")  # GSLS_LIB: A/B builds

c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_void_p = ctypes.c_void_p

# status codes (gsls_status_t)
OK, ERR_ARG, ERR_CUDA, ERR_SINGULAR, ERR_ILL, ERR_CACHE, ERR_NONFINITE, ERR_TOO_LARGE, ERR_NO_DEVICE = range(9)
ERR_LOWRANK = 9  # internal: a factored combine met an indefinite P; the scan re-runs dense (include/gsls.h)


class Dims(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("nu", ctypes.c_int32), ("nc", ctypes.c_int32),
                ("nf", ctypes.c_int32), ("N", ctypes.c_int32), ("batch", ctypes.c_int32)]


QP_FIELDS = ("A", "B", "b", "Q", "R", "S", "q", "r", "QN", "qN", "C", "D", "f", "CN", "fN", "dx0")


class Qp(ctypes.Structure):
    _fields_ = [(k, c_void_p) for k in QP_FIELDS]


class AdmmSettings(ctypes.Structure):
    _fields_ = [("rho0", ctypes.c_double), ("rho_min", ctypes.c_double), ("rho_max", ctypes.c_double),
                ("sigma", ctypes.c_int32), ("tol_primal", ctypes.c_double), ("tol_dual", ctypes.c_double),
                ("max_iter", ctypes.c_int32)]


class AdmmState(ctypes.Structure):
    _fields_ = [("z", c_void_p), ("lam", c_void_p), ("y", c_void_p), ("rho", c_void_p),
                ("r_primal", c_void_p), ("r_dual", c_void_p), ("generation", c_void_p),
                ("iteration", c_void_p)]


class AdmmStats(ctypes.Structure):
    _fields_ = [("iterations", c_void_p), ("converged", c_void_p), ("rho_changes", c_void_p),
                ("cache_builds", c_void_p)]


class LinArgs(ctypes.Structure):
    _fields_ = [("model_id", ctypes.c_int32), ("params", c_void_p), ("cons_offset", ctypes.c_int32),
                ("x", c_void_p), ("u", c_void_p), ("h", c_void_p), ("hf", c_void_p), ("xbar0", c_void_p),
                ("Qw", c_void_p), ("Rw", c_void_p), ("QNw", c_void_p), ("xref", c_void_p), ("uref", c_void_p),
                ("E_const", c_void_p), ("write_weights", ctypes.c_int32)]


class RtiStepArgs(ctypes.Structure):
    """gsls_rti_step_args_t (include/gsls.h)."""
    _fields_ = ([("lin", LinArgs), ("qp", ctypes.POINTER(Qp)), ("E", c_void_p), ("E_in", c_void_p)]
                + [(k, ctypes.c_int32) for k in ("robust", "use_tau", "warm_admm", "no_overlap")]
                + [(k, c_void_p) for k in ("Qbar", "Rbar", "QbarN", "tau", "tau_term", "beta", "beta_term")]
                + [("eps", ctypes.c_double), ("admm", AdmmSettings), ("state", AdmmState), ("stats", AdmmStats)]
                + [(k, c_void_p) for k in ("h", "hf", "dx", "du", "plan_x", "plan_u", "warm_x", "warm_u", "u0",
                                           "cost")])


class RolloutArgs(ctypes.Structure):
    _fields_ = [("model_id", ctypes.c_int32), ("params", c_void_p), ("cons_offset", ctypes.c_int32),
                ("x", c_void_p), ("u", c_void_p), ("phi_u", c_void_p), ("E", c_void_p), ("E_pinv", c_void_p),
                ("disturbances", c_void_p), ("h", c_void_p), ("tol_lin", ctypes.c_double),
                ("rollouts", ctypes.c_int32)]


class RolloutOut(ctypes.Structure):
    _fields_ = [(k, c_void_p) for k in ("x", "u", "w", "stage_g", "terminal_g", "tube_margin", "max_w_norm",
                                        "flags")]


class Error(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("instance", ctypes.c_int32), ("where", ctypes.c_int32),
                ("aux", ctypes.c_int32), ("aux2", ctypes.c_int32), ("message", ctypes.c_char * 256)]


_SIGS = {
    "gsls_version": ([], ctypes.c_int),
    "gsls_last_error": ([ctypes.POINTER(Error)], ctypes.c_int),
    "gsls_ctx_create": ([ctypes.POINTER(Dims), ctypes.POINTER(c_void_p)], ctypes.c_int),
    "gsls_ctx_destroy": ([c_void_p], ctypes.c_int),
    "gsls_ctx_bytes": ([c_void_p], ctypes.c_int64),
    "gsls_ctx_check": ([c_void_p, c_void_p], ctypes.c_int),
    "gsls_scan_plan": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_int32_p, c_int32_p, c_int32_p,
                        c_int32_p, c_int32_p], ctypes.c_int),
    "gsls_lqr_solve": ([c_void_p, ctypes.POINTER(Qp), ctypes.c_int32] + [c_void_p] * 6 + [c_void_p], ctypes.c_int),
    "gsls_lqr_solve_cached": ([c_void_p, ctypes.POINTER(Qp), c_void_p, c_void_p, c_void_p, ctypes.c_int32]
                              + [c_void_p] * 4 + [c_void_p], ctypes.c_int),
    "gsls_admm_solve_qp": ([c_void_p, ctypes.POINTER(Qp), ctypes.POINTER(AdmmSettings),
                            ctypes.POINTER(AdmmState), ctypes.POINTER(AdmmStats), c_void_p, c_void_p,
                            c_void_p], ctypes.c_int),
    "gsls_ctx_export_solution": ([c_void_p] * 6, ctypes.c_int),
    "gsls_admm_build_cache": ([c_void_p, ctypes.POINTER(Qp), c_void_p, c_void_p], ctypes.c_int),
    "gsls_sls_ncell": ([ctypes.c_int32], ctypes.c_int),
    "gsls_sls_set_columns": ([c_void_p, ctypes.c_int32, ctypes.c_int32], ctypes.c_int),
    "gsls_sls_plan": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_int32] + [c_int32_p] * 6, ctypes.c_int),
    "gsls_sls_assemble": ([c_void_p, ctypes.POINTER(Qp)] + [c_void_p] * 5 + [ctypes.c_int32, c_void_p], ctypes.c_int),
    "gsls_sls_set_costs": ([c_void_p] * 5, ctypes.c_int),
    "gsls_sls_export_costs": ([c_void_p] * 5, ctypes.c_int),
    "gsls_sls_synthesize": ([c_void_p, ctypes.POINTER(Qp), c_void_p, c_void_p], ctypes.c_int),
    "gsls_sls_tighten": ([c_void_p, ctypes.POINTER(Qp), c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "gsls_sls_duals": ([c_void_p, ctypes.POINTER(Qp), c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int32]
                       + [c_void_p] * 5, ctypes.c_int),
    "gsls_sls_import_response": ([c_void_p] * 4, ctypes.c_int),
    "gsls_sls_export": ([c_void_p] * 5, ctypes.c_int),
    "gsls_sls_cost": ([c_void_p] * 6, ctypes.c_int),
    "gsls_linearize": ([c_void_p, ctypes.POINTER(LinArgs), ctypes.POINTER(Qp), c_void_p, c_void_p], ctypes.c_int),
    "gsls_traj_eval": ([c_void_p, ctypes.POINTER(LinArgs), c_void_p, c_void_p], ctypes.c_int),
    "gsls_apply_tightening": ([c_void_p] * 6, ctypes.c_int),
    "gsls_prof_enable": ([ctypes.c_int32], ctypes.c_int),
    "gsls_prof_read": ([c_void_p, c_void_p, c_void_p, ctypes.c_int32], ctypes.c_int),
    "gsls_rti_apply": ([c_void_p] * 17, ctypes.c_int),
    "gsls_rti_step": ([c_void_p, ctypes.POINTER(RtiStepArgs), c_void_p], ctypes.c_int),
    "gsls_rti_pack_results": ([c_void_p, c_void_p, ctypes.POINTER(AdmmStats), c_void_p, c_void_p, c_void_p],
                              ctypes.c_int),
    "gsls_rollout": ([c_void_p, ctypes.POINTER(RolloutArgs), ctypes.POINTER(RolloutOut), c_void_p], ctypes.c_int),
}

PROF_FAMILIES = ("leaf", "cvf_lqr", "gains", "cot", "replay", "sls_assemble", "sls_leaf", "sls_cvf", "sls_gains",
                 "sls_matprod", "sls_phiu", "sls_rownorm", "sls_small", "linearize", "rti_misc", "rollout")

# every symbol include/gsls.h declares (checked by the CPU test suite)
EXPORTS = tuple(_SIGS)

_lib = None


def load(require_device: bool = True):
    """Load libgsls.so (raises when missing; no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                               "(the GPU-SLS path has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    if require_device:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("the GPU-SLS path needs a CUDA device (no CPU fallback)")
    return _lib


def last_error() -> Error:
    e = Error()
    load(False).gsls_last_error(ctypes.byref(e))
    return e


def check(rc: int, what: str = "gsls call"):
    """Map a gsls_status_t to the reference's exception classes."""
    if rc == OK:
        return
    from . import errors
    e = last_error()
    msg = e.message.decode(errors="replace") or what
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_SINGULAR:
        raise errors.SingularStageError(msg)
    if rc == ERR_ILL:
        raise errors.IllConditionedCombineError(msg)
    if rc == ERR_CACHE:
        raise errors.CacheInvalidatedError(msg)
    if rc == ERR_NONFINITE:
        raise ArithmeticError(msg)
    raise RuntimeError(f"{what}: {msg} (status {rc})")
