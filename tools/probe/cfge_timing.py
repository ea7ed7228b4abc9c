"""cfg-E (75D/19u humanoid, N = 2047: 192,493 variables, 81,882 constraints) admm.solve_qp
through the drop-in API: wall time and ADMM stats, plus the replay family's device time.

    python tools/probe/cfge_timing.py
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2604_07644_b200 import _native as nat, admm, scenarios as S, sqp  # noqa: E402

me = S.cfge_model()
N = S.CFGE["N"]
x, u = S.cfge_trajectory(me, N)
qp = sqp.linearize(me, sqp.Trajectory(x, u, me.dt), None, S.cfge_start(me))
st = admm.AdmmSettings(**S.CFGE["admm"])
r = admm.solve_qp(qp, st)
lib = nat.load()
for rep in range(2):
    torch.cuda.synchronize()
    lib.gsls_prof_enable(1)
    lib.gsls_prof_read(None, None, None, 0)
    t = time.perf_counter()
    r = admm.solve_qp(qp, st)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    lib.gsls_prof_enable(0)
    nfam = len(nat.PROF_FAMILIES)
    pm, pl = np.zeros(nfam), np.zeros(nfam, np.int64)
    lib.gsls_prof_read(pm.ctypes.data, None, pl.ctypes.data, nfam)
    fam = {k: round(float(v), 3) for k, v, c in zip(nat.PROF_FAMILIES, pm, pl) if c}
    print(f"cfg-E solve_qp: {ms:.1f} ms wall, iterations {r.stats.iterations}, builds {r.stats.cache_builds}, "
          f"converged {r.stats.converged}; device ms by family {fam}", flush=True)
