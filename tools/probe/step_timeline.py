"""Per-phase device time of one batched robust RTI step (cfg-D), streams serialized
(GSLS_OVERLAP=0) so the phases add up, plus the ADMM's rebuild waves (GSLS_ADMM_VERBOSE).

    python tools/probe/step_timeline.py [--batch B] [--tag q61]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("GSLS_OVERLAP", "0")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_07644_b200 import _native as nat, scenarios as S  # noqa: E402
from paper_2604_07644_b200.engine import RtiEngine  # noqa: E402
from paper_2604_07644_b200.sls import ragged_to_cells  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--tag", default="q61")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    wl = S.rti_workload(a.tag)
    m, N, B = wl.model, wl.N, a.batch
    eng = RtiEngine(m, N, B, S.our_settings()(m))
    d = lambda x: torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")  # noqa: E731
    xs = d(wl.scenario_states(0, B))
    px = d(np.broadcast_to(wl.prev_x, (B,) + wl.prev_x.shape))
    pu = d(np.broadcast_to(wl.prev_u, (B,) + wl.prev_u.shape))
    tc = d(np.broadcast_to(ragged_to_cells(wl.tau, N, (m.nc,)), (B, N * (N + 1) // 2, m.nc)))
    tt = d(np.broadcast_to(wl.tau_term, (B, N, m.nf)))
    eng.step(xs, px, pu, tau=tc, tau_term=tt)
    torch.cuda.synchronize()
    lib = nat.load()
    lib.gsls_prof_enable(1)
    lib.gsls_prof_read(None, None, None, 0)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        eng.step(xs, px, pu, tau=tc, tau_term=tt)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / a.steps * 1e3
    lib.gsls_prof_enable(0)
    nf = len(nat.PROF_FAMILIES)
    ms, un, nl = np.zeros(nf), np.zeros(nf), np.zeros(nf, np.int64)
    lib.gsls_prof_read(ms.ctypes.data, un.ctypes.data, nl.ctypes.data, nf)
    its = eng.stats.iterations.cpu().numpy()
    print(f"B={B} {a.tag}: wall {wall:.2f} ms/step (serialized streams); ADMM iterations mean {its.mean():.1f} "
          f"max {its.max()} sum {its.sum()}; rho changes {eng.stats.rho_changes.cpu().numpy().sum()}")
    q = np.percentile(its, [10, 50, 90, 99])
    print(f"  iterations p10/p50/p90/p99 {q.tolist()}; histogram (25-wide bins): "
          f"{np.bincount(its // 25).tolist()}")
    tot = 0.0
    for k, v, c in zip(nat.PROF_FAMILIES, ms, nl):
        if c:
            tot += v / a.steps
            print(f"  {k:14s} {v / a.steps:9.3f} ms  {c // a.steps:5d} launches")
    print(f"  {'sum':14s} {tot:9.3f} ms")


if __name__ == "__main__":
    main()
