"""SLS synthesis (sls.py:227-318) through the product API vs the float64 oracle on random
problems of several shapes; run under GSLS_LOWRANK=0 and the default to compare the dense
and factored combine trees shape by shape.

    python tools/probe/sls_factored_shapes.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import sls as osls  # noqa: E402
from paper_2604_07644_b200 import sls  # noqa: E402


def case(nx, nu, N, c, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, nx, nx)) * 0.3 + np.eye(nx)
    A /= np.linalg.norm(A, 2, axis=(1, 2), keepdims=True)
    B = rng.standard_normal((N, nx, nu)) * 0.5
    E = rng.standard_normal((N, nx, nx)) * 0.05
    C = rng.standard_normal((N, c, nx))
    D = rng.standard_normal((N, c, nu))
    CN = rng.standard_normal((2, nx))
    oc = osls.assemble_costs(None, C, D, CN, osls.Weights.identity(nx, nu))
    ref = osls.synthesize(A, B, E, oc)
    got = sls.synthesize(A, B, E, sls.SlsCosts(oc.Qx, oc.Qu, oc.Qux, oc.Qx_term))
    ex = max(oracle.relative_error(got.Phi_x[j], ref.Phi_x[j]) for j in range(N))
    eg = max(oracle.relative_error(got.gains[j], ref.gains[j]) for j in range(N) if len(ref.gains[j]))
    return ex, eg


for shp in [(4, 2, 20, 4), (6, 3, 12, 4), (12, 4, 20, 6), (12, 4, 50, 13), (16, 4, 30, 6), (20, 8, 25, 6),
            (32, 8, 25, 8), (61, 12, 25, 26), (75, 19, 12, 8)]:
    ex, eg = case(*shp, seed=1)
    print(f"nx={shp[0]:2d} nu={shp[1]:2d} N={shp[2]:2d}: Phi_x {ex:.2e} gains {eg:.2e}", flush=True)
