"""Repeated robust RTI steps (engine-held duals carried over) at batch 1 vs batch B:
instance 0 must follow the same path, and the float64 oracle's step sequence.

    python tools/probe/multistep_batch.py [B] [steps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2604_07644_b200 import scenarios as S  # noqa: E402
from paper_2604_07644_b200.engine import RtiEngine  # noqa: E402
from paper_2604_07644_b200.sls import ragged_to_cells  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = S.rti_workload("q61")
m, N = wl.model, wl.N
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")  # noqa: E731


def run(Bx):
    rep = lambda a: np.broadcast_to(a, (Bx,) + np.shape(a))  # noqa: E731
    e = RtiEngine(m, N, Bx, S.our_settings()(m))
    xb, px, pu = d(wl.scenario_states(0, Bx)), d(rep(wl.prev_x)), d(rep(wl.prev_u))
    tc, tt = d(rep(ragged_to_cells(wl.tau, N, (m.nc,)))), d(rep(wl.tau_term))
    out = []
    for k in range(steps):
        if k == 0:
            e.step(xb, px, pu, tau=tc, tau_term=tt)
        else:
            e.step(xb, px, pu)
        torch.cuda.synchronize()
        out.append((int(e.stats.iterations[0]), e.u0[0].cpu().numpy().copy(), e.tau[0].cpu().numpy().copy()))
    return out


if os.environ.get("ORDER") == "b1":
    rb, r1 = run(B), run(1)
else:
    r1, rb = run(1), run(B)
import test_oracle_golden  # noqa: E402,F401
from bench import oracle_settings  # noqa: E402
rs = oracle_settings(m)
tau = oracle.sls.Duals.zero(N, m.nc, m.nf, rs.eps)
tau.tau, tau.tau_term = wl.tau, wl.tau_term
prev = oracle.sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
x = wl.scenario_states(0, 1)[0]
for k in range(steps):
    r = oracle.sls.rti_robust_step(m, x, prev, tau, rs)
    tau = r.tau
    print(f"step {k}: oracle its {r.stats.admm_iterations}; B=1 its {r1[k][0]} u0 err "
          f"{oracle.relative_error(r1[k][1], r.u0):.2e}; B={B} inst0 its {rb[k][0]} u0 err "
          f"{oracle.relative_error(rb[k][1], r.u0):.2e}; B1 vs B tau equal {np.array_equal(r1[k][2], rb[k][2])}",
          flush=True)
