"""How sensitive are the chained SQP / robust solves of cfg-B and cfg-C to perturbations
far below float32 resolution?  Runs the float64 oracle (pinned to the reference) on the
benchmark inputs and on copies whose initial trajectory is perturbed by eps (absolute,
seeded normal noise), and reports the largest change of every output the GPU tests
compare.  A change above the 1e-4 bar (or of an iteration count) at eps = 1e-7 means the
float64 reference itself does not determine that output to the bar's precision.

    python tools/probe/chain_sensitivity.py [cfgb|cfgc] [eps ...]
    python tools/probe/chain_sensitivity.py midchain   # perturb the trajectory at QP call k
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import admm as oadmm, sls as osls, sqp as osqp  # noqa: E402
from paper_2604_07644_b200 import scenarios as S  # noqa: E402


def run(which, eps, seed=0):
    calls = []
    orig = oadmm.solve_qp

    def wrap(*a, **k):
        r = orig(*a, **k)
        calls.append(r.stats.iterations)
        return r
    osqp.admm.solve_qp = wrap
    try:
        rng = np.random.default_rng(seed)
        cfg = S.CFGB if which == "cfgb" else S.CFGC
        m = S.cfgb_model() if which == "cfgb" else S.cfgc_model()
        x0 = S.quad12_start()
        xg, ug = S.hover_guess(m, x0, cfg["N"])
        if eps:
            xg = xg + eps * rng.standard_normal(xg.shape)
            ug = ug + eps * rng.standard_normal(ug.shape)
        st = osqp.Settings(admm=oadmm.Settings(**cfg["admm"]), **cfg["sqp"])
        init = osqp.Trajectory(xg, ug, m.dt)
        if which == "cfgb":
            r = osqp.solve_nmpc(m, x0, st, init)
            out = {"x": r.trajectory.x, "u": r.trajectory.u, "lam_s": r.lam_stage, "lam_t": r.lam_terminal,
                   "sqp_iters": r.stats.iterations}
        else:
            rs = osls.RobustSettings(sqp=st, weights=osls.Weights.identity(m.nx, m.nu), eps=cfg["eps"],
                                     tol_h=cfg["tol_h"], max_alternations=cfg["max_alternations"])
            r = osls.solve_robust(m, x0, rs, initial=init)
            out = {"x": r.trajectory.x, "h": r.tightening.h, "lam_s": r.lam_stage, "tau_term": r.duals.tau_term,
                   "alternations": r.stats.alternations, "sqp_iters": r.stats.sqp_iterations}
        out["qp_iters"] = np.array(calls)
        return out
    finally:
        osqp.admm.solve_qp = orig


def midchain(which="cfgb", calls_to_probe=(3, 4), epss=(1e-8, 1e-7, 1e-6), trials=4):
    """Re-solve inner QP call k of the float64 SQP from a trajectory perturbed by eps (the
    reference's own warm ADMM state and settings): does the iteration count move?"""
    import copy
    cfg = S.CFGB
    m = S.cfgb_model()
    x0 = S.quad12_start()
    xg, ug = S.hover_guess(m, x0, cfg["N"])
    st = osqp.Settings(admm=oadmm.Settings(**cfg["admm"]), **cfg["sqp"])
    trajs, calls = [], []
    lin0, qp0 = osqp.linearize, oadmm.solve_qp

    def lin(model, traj, *a, **k):
        trajs.append(copy.deepcopy(traj))
        return lin0(model, traj, *a, **k)

    def qp(q, s, warm_start=None, **k):
        calls.append((s, copy.deepcopy(warm_start)))
        return qp0(q, s, warm_start=warm_start, **k)
    osqp.linearize, osqp.admm.solve_qp = lin, qp
    try:
        osqp.solve_nmpc(m, x0, st, osqp.Trajectory(xg, ug, m.dt))
    finally:
        osqp.linearize, osqp.admm.solve_qp = lin0, qp0
    rng = np.random.default_rng(0)
    for i in calls_to_probe:
        s, w = calls[i]
        tr = trajs[i]
        base = qp0(lin0(m, tr, None, x0), s, warm_start=copy.deepcopy(w)).stats.iterations
        for eps in epss:
            its = []
            for _ in range(trials):
                t2 = osqp.Trajectory(tr.x + eps * rng.standard_normal(tr.x.shape),
                                     tr.u + eps * rng.standard_normal(tr.u.shape), tr.dt)
                its.append(qp0(lin0(m, t2, None, x0), s, warm_start=copy.deepcopy(w)).stats.iterations)
            print(f"  {which} QP call {i}: unperturbed {base} iterations; trajectory + {eps:g} noise: {its}",
                  flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "midchain":
        midchain()
        return
    which = sys.argv[1] if len(sys.argv) > 1 else "cfgb"
    epss = [float(e) for e in sys.argv[2:]] or [1e-9, 1e-7]
    base = run(which, 0.0)
    print(f"{which}: float64 oracle, unperturbed: qp iterations {base['qp_iters'].tolist()}")
    for eps in epss:
        for seed in range(2):
            o = run(which, eps, seed)
            rep = []
            for k, v in base.items():
                if k == "qp_iters":
                    same = o[k].shape == v.shape
                    d = int(np.abs(o[k] - v).max()) if same else "different length"
                    rep.append(f"qp_iters max|d|={d}")
                elif np.ndim(v) == 0:
                    rep.append(f"{k} {o[k]} vs {v}")
                else:
                    rep.append(f"{k} rel={oracle.relative_error(o[k], v):.2e}")
            print(f"  eps={eps:g} seed={seed}: " + "; ".join(rep), flush=True)


if __name__ == "__main__":
    main()
