"""Batched robust RTI step (cfg-D, B = 1024 by default): eager RtiEngine.step vs one
CUDA-graph launch (RtiEngine.capture: the ADMM as a conditional WHILE node over
[rebuild | persistent replay | decide]), device time per step and iteration parity.

    python tools/probe/graph_batch.py [batch] [steps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2604_07644_b200 import scenarios as S  # noqa: E402
from paper_2604_07644_b200.engine import RtiEngine  # noqa: E402
from paper_2604_07644_b200.sls import ragged_to_cells  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = S.rti_workload("q61")
m, N = wl.model, wl.N
d = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")  # noqa: E731
xs = d(wl.scenario_states(0, B))
px = d(np.broadcast_to(wl.prev_x, (B,) + wl.prev_x.shape))
pu = d(np.broadcast_to(wl.prev_u, (B,) + wl.prev_u.shape))
tc = d(np.broadcast_to(ragged_to_cells(wl.tau, N, (m.nc,)), (B, N * (N + 1) // 2, m.nc)))
tt = d(np.broadcast_to(wl.tau_term, (B, N, m.nf)))


def timed(fn):
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


eng = RtiEngine(m, N, B, S.our_settings()(m))
eager = timed(lambda: eng.step(xs, px, pu, tau=tc, tau_term=tt))
its_e = eng.stats.iterations.cpu().numpy().copy()
g = eng.capture(xs, px, pu)
graph = timed(lambda: g())
g.check()
its_g = eng.stats.iterations.cpu().numpy().copy()
print(f"B={B}: eager {eager:.2f} ms/step, graph {graph:.2f} ms/step; iterations equal {np.array_equal(its_e, its_g)} "
      f"(mean {its_e.mean():.1f} / {its_g.mean():.1f})")
