"""Device vs reference per-QP ADMM iteration counts of the cfg-B SQP (tests/golden/cfgb.npz)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle
from conftest import load_golden
from paper_2604_07644_b200 import admm, scenarios as S, sqp
g = load_golden("cfgb")
m = S.cfgb_model(); N = S.CFGB["N"]; x0 = S.quad12_start()
xg, ug = S.hover_guess(m, x0, N)
st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGB["admm"]), **S.CFGB["sqp"])
r = sqp.solve_nmpc(m, x0, st, sqp.Trajectory(xg, ug, m.dt))
print("device   ", [c[0] for c in r.stats.qp_calls])
print("reference", g["qp_calls"][:, 0].tolist())
print("sqp iters", r.stats.iterations, int(g["sqp_iters"]), "x rel", oracle.relative_error(r.trajectory.x, g["x"]),
      "lam rel", oracle.relative_error(r.lam_stage, g["lam_s"]), "residual", r.stats.residual, float(g["residual"]))
