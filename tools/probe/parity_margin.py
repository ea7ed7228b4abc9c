"""Worst relative errors (reference.relative_error) of the benched batch against the real
reference's fixture (tests/golden/batch.npz): how much of the 1e-4 bar each field uses.

    python tools/probe/parity_margin.py
"""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from test_gpu_batch import _engine_step, _host
from conftest import load_golden
import oracle, problems as P
from paper_2604_07644_b200.sls import cells_to_ragged
g = load_golden("batch")
for tag, count in (("q61", 64), ("h75", 16)):
    eng, wl, xs = _engine_step(tag, count)
    m, N = wl.model, wl.N
    tau = _host(eng.tau)
    worst = {}
    for i in range(count):
        for k, a, b in (("u0", _host(eng.u0[i]), g[f"{tag}_u0"][i]), ("h", _host(eng.h[i]), g[f"{tag}_h"][i]),
                        ("lam", _host(eng.state.lam[i]), g[f"{tag}_lam"][i].astype(float)),
                        ("tau", P.pack_lower(cells_to_ragged(tau[i], N, 1, N), N, 1, N, (m.nc,)), g[f"{tag}_tau"][i].astype(float)),
                        ("tau_term", _host(eng.tau_term[i]), g[f"{tag}_tau_term"][i])):
            e = oracle.relative_error(a, b)
            if e > worst.get(k, (0, -1))[0]: worst[k] = (e, i)
    print(tag, {k: (f"{v[0]:.3g}", v[1]) for k, v in worst.items()})
