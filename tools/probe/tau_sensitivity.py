"""Where does the batched robust step's tau deviate from the reference fixture?

tau = lambda_k / sqrt(beta + eps) (sls.py:150-173) amplifies the ADMM dual's absolute
error by 1/sqrt(beta + eps) where beta is small.  Prints, per instance, the relative
errors of lambda and tau, and at the worst tau entry: beta, lambda (ours / reference).

    python tools/probe/tau_sensitivity.py [q61|h75] [count]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import problems as P  # noqa: E402
from conftest import load_golden  # noqa: E402
from test_gpu_batch import _engine_step, _host  # noqa: E402


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "q61"
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    g = load_golden("batch")
    eng, wl, xs = _engine_step(tag, count)
    m, N = wl.model, wl.N
    from paper_2604_07644_b200.sls import cells_to_ragged
    tau = _host(eng.tau)
    beta = _host(eng.beta)
    worst = []
    for i in range(count):
        t_ours = P.pack_lower(cells_to_ragged(tau[i], N, 1, N), N, 1, N, (m.nc,))
        b_ours = P.pack_lower(cells_to_ragged(beta[i], N, 1, N), N, 1, N, (m.nc,))
        t_ref = g[f"{tag}_tau"][i].astype(float)
        et = oracle.relative_error(t_ours, t_ref)
        el = oracle.relative_error(_host(eng.state.lam[i]), g[f"{tag}_lam"][i].astype(float))
        d = np.abs(t_ours - t_ref)
        idx = np.unravel_index(np.argmax(d), d.shape)
        worst.append(et)
        lam_i = _host(eng.state.lam[i])
        print(f"inst {i:2d}: lam {el:.2e} tau {et:.2e} (max|tau| {np.abs(t_ref).max():.3g}) at {idx}: "
              f"tau {t_ours[idx]:.6g} vs {t_ref[idx]:.6g}, beta {b_ours[idx]:.3g}")
    print("worst tau", max(worst), "instances over 1e-4:", sum(w > 1e-4 for w in worst))


if __name__ == "__main__":
    main()
