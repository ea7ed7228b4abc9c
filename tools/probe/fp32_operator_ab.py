"""A/B: ADMM iteration counts of the cfg-B SQP's inner QPs with float64 operators (the
reference / oracle), with every cached operator rounded to float32 (the device's storage
precision, vector recursion still float64: an emulation on the CPU) and on the device.

    python tools/probe/fp32_operator_ab.py            # CPU columns only
    python tools/probe/fp32_operator_ab.py --device   # adds the device column (GPU box)

Each QP call k is re-solved from the warm ADMM state the reference passed in, so the
columns differ only in the precision of the cached factorization."""
import copy
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from oracle import admm as oadmm, lqr as olqr, sqp as osqp  # noqa: E402
from paper_2604_07644_b200 import scenarios as S  # noqa: E402


def _round(x):
    if isinstance(x, np.ndarray) and x.dtype == np.float64:
        return x.astype(np.float32).astype(np.float64)
    if isinstance(x, (list, tuple)):
        return type(x)(_round(v) for v in x)
    if isinstance(x, dict):
        return {k: _round(v) for k, v in x.items()}
    return x


def fp32_operators():
    """Patch oracle.lqr.build_cache so every recorded operator is rounded to float32."""
    orig = olqr.build_cache

    def build(qp, generation=0):
        sol, cache = orig(qp, generation)
        for f in ("stat", "K", "Gamma", "P", "Abar", "cvf_tape", "cot_tape"):
            setattr(cache, f, _round(getattr(cache, f)))
        return sol, cache
    olqr.build_cache = build
    oadmm.lqr.build_cache = build
    return orig


def main(device: bool):
    m = S.cfgb_model()
    N = S.CFGB["N"]
    x0 = S.quad12_start()
    xg, ug = S.hover_guess(m, x0, N)
    st = osqp.Settings(admm=oadmm.Settings(**S.CFGB["admm"]), **S.CFGB["sqp"])
    calls = []
    orig = oadmm.solve_qp

    def wrap(qp, s, warm_start=None, **k):
        calls.append((qp, s, copy.deepcopy(warm_start)))
        return orig(qp, s, warm_start=warm_start, **k)
    osqp.admm.solve_qp = wrap
    osqp.solve_nmpc(m, x0, st, osqp.Trajectory(xg, ug, m.dt))
    osqp.admm.solve_qp = orig
    f64 = [orig(qp, s, warm_start=copy.deepcopy(w)).stats.iterations for qp, s, w in calls]
    b = fp32_operators()
    f32 = [orig(qp, s, warm_start=copy.deepcopy(w)).stats.iterations for qp, s, w in calls]
    olqr.build_cache = oadmm.lqr.build_cache = b
    dev = [None] * len(calls)
    if device:
        from paper_2604_07644_b200 import admm
        for i, (qp, s, w) in enumerate(calls):
            ws = None
            if w is not None:
                ws = admm.AdmmState(z=w.z.copy(), lam=w.lam.copy(), y=w.y.copy(), rho=w.rho,
                                    generation=w.generation, iteration=w.iteration)
            dev[i] = admm.solve_qp(qp, admm.AdmmSettings(rho0=s.rho0, rho_min=s.rho_min, rho_max=s.rho_max,
                                                         sigma=s.sigma, tol_primal=s.tol_primal,
                                                         tol_dual=s.tol_dual, max_iter=s.max_iter),
                                   warm_start=ws).stats.iterations
    print("call  float64  float32-operators(emulated)  device")
    for i in range(len(calls)):
        print(f"{i:4d}  {f64[i]:7d}  {f32[i]:27d}  {dev[i]}")


if __name__ == "__main__":
    main("--device" in sys.argv)
