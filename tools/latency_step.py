"""Runs single-instance robust RTI steps (bench latency workload) for ncu captures.

    python tools/latency_step.py [q61|h75] [steps] [batch]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07644_b200 import scenarios  # noqa: E402
from paper_2604_07644_b200.engine import RtiEngine  # noqa: E402
from paper_2604_07644_b200.sls import ragged_to_cells  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "q61"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
wl = scenarios.rti_workload(tag)
m = wl.model
eng = RtiEngine(m, wl.N, B, scenarios.our_settings()(m))
d = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
rep = lambda a: np.broadcast_to(a, (B,) + np.shape(a)).copy()  # noqa: E731
xb, px, pu = d(wl.scenario_states(0, B)), d(rep(wl.prev_x)), d(rep(wl.prev_u))
tc, tt = d(rep(ragged_to_cells(wl.tau, wl.N, (m.nc,)))), d(rep(wl.tau_term))
times = []
for _ in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step(xb, px, pu, tau=tc, tau_term=tt)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
print(tag, "cluster", os.environ.get("GSLS_REPLAY_CLUSTER", "auto"), "iterations", int(eng.stats.iterations[0]),
      "u0", eng.u0[0, :3].tolist(), "ms", sorted(times)[len(times) // 2])
