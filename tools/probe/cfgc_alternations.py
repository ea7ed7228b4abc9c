"""cfg-C solve_robust (sls.py:400-469): per-alternation dh and synthesis checks, to compare
combine variants (GSLS_LOWRANK) against the reference fixture (tests/golden/cfgc.npz).

    GSLS_LOWRANK=0 python tools/probe/cfgc_alternations.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden  # noqa: E402
from paper_2604_07644_b200 import admm, scenarios as S, sls, sqp  # noqa: E402

g = load_golden("cfgc")
m = S.cfgc_model()
N = S.CFGC["N"]
x0 = S.quad12_start()
xg, ug = S.hover_guess(m, x0, N)
st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGC["admm"]), **S.CFGC["sqp"])
rs = sls.RobustSettings(sqp=st, weights=sls.SlsWeights.identity(m.nx, m.nu), eps=S.CFGC["eps"],
                        tol_h=S.CFGC["tol_h"], max_alternations=S.CFGC["max_alternations"])
orig = sls.tighten
prev = [None]


def traced(resp, C, D, CN, executor=None):
    t = orig(resp, C, D, CN, executor=executor)
    dh = t.max_abs_diff(prev[0]) if prev[0] is not None else float("inf")
    print(f"  alternation: max h {np.abs(t.h).max():.6f} dh {dh:.3e}", flush=True)
    prev[0] = t
    return t


sls.tighten = traced
r = sls.solve_robust(m, x0, rs, initial=sqp.Trajectory(xg, ug, m.dt))
print("ours:", r.stats, "ref alternations", int(g["alternations"]), "sqp", int(g["sqp_iters"]))
