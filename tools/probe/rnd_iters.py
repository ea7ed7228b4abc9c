"""Probe: ADMM iteration counts of the reference's random fixtures (tol 1e-6) on the device."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import admm as oadmm, lqr as olqr
from conftest import load_golden
from paper_2604_07644_b200 import admm
g = load_golden("admm")
for i in range(3):
    qp = olqr.QP(**{k: g[f"rnd{i}_qp_{k}"] for k in olqr.FIELDS})
    res = admm.solve_qp(qp, admm.AdmmSettings(tol_primal=1e-6, tol_dual=1e-6))
    f = oadmm.offsets(qp)
    ref = oadmm.solve_qp(qp, oadmm.Settings(tol_primal=1e-6, tol_dual=1e-6))
    print(i, "device", res.stats.iterations, "golden", int(g[f"rnd{i}_iters"]), "rho_changes", res.stats.rho_changes,
          "active eq", bool(((res.state.z >= f - 1e-12) == (ref.state.z >= f - 1e-12)).all()),
          "rp", res.state.r_primal, "rd", res.state.r_dual)
