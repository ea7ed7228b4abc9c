"""CPU check of the merged SLS column schedules (csrc/sls.cu merge_columns):
executing them in float64 numpy with the oracle's combine reproduces the
reference grid synthesis (tests/golden/sls.npz), so the neutral-element
elision and the triangular cell layout are exact.  No kernel launches."""

import ctypes

import numpy as np
import pytest

from conftest import load_golden
from oracle import lqr as olqr, sls as osls
from paper_2604_07644_b200 import _native as nat
from paper_2604_07644_b200.sls import cell_index, cells_to_ragged, ragged_to_cells

I32 = ctypes.POINTER(ctypes.c_int32)


def sls_plan(N, cvf):
    lib = nat.load(require_device=False)
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    z = np.zeros(1, np.int32)
    nat.check(lib.gsls_sls_plan(N, cvf, 0, z.ctypes.data_as(I32), z.ctypes.data_as(I32), z.ctypes.data_as(I32),
                                ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    ops = np.zeros((a.value, 3), np.int32)
    lo = np.zeros(b.value + 1, np.int32)
    out = np.zeros(N * (N + 1) // 2, np.int32)
    nat.check(lib.gsls_sls_plan(N, cvf, a.value, ops.ctypes.data_as(I32), lo.ctypes.data_as(I32),
                                out.ctypes.data_as(I32), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return ops, lo, out, c.value


def emulate(A, B, E, costs):
    N, n = A.shape[0], A.shape[-1]
    ops, _, out, ns = sls_plan(N, 1)
    P, Am, Cm = [None] * ns, [None] * ns, [None] * ns
    for j in range(N):
        for k in range(j + 1, N + 1):
            c = cell_index(N, k, j)
            if k == N:
                P[c], Am[c], Cm[c] = costs.Qx_term[j], np.zeros((n, n)), np.zeros((n, n))
            else:
                Qx, Qu, Qux = costs.Qx[j][k - j - 1], costs.Qu[j][k - j - 1], costs.Qux[j][k - j - 1]
                Qi = np.linalg.inv(Qu)
                P[c], Am[c], Cm[c] = Qx - Qux.T @ Qi @ Qux, A[k] - B[k] @ Qi @ Qux, B[k] @ Qi @ B[k].T
    for d, e, l in ops:
        r = olqr.cvf_matrix(P[e][None], Am[e][None], Cm[e][None], P[l][None], Am[l][None], Cm[l][None])
        P[d], Am[d], Cm[d] = r[0][0], r[1][0], r[2][0]
    mops, _, mout, mns = sls_plan(N, 0)
    M = [None] * mns
    for j in range(N):
        M[cell_index(N, j + 1, j)] = E[j]
        for k in range(j + 1, N):
            Pn = P[out[cell_index(N, k + 1, j)]]
            Qu, Qux = costs.Qu[j][k - j - 1], costs.Qux[j][k - j - 1]
            K = -np.linalg.inv(Qu + B[k].T @ Pn @ B[k]) @ (Qux + B[k].T @ Pn @ A[k])
            M[cell_index(N, k + 1, j)] = A[k] + B[k] @ K
    for d, e, l in mops:
        M[d] = M[l] @ M[e]
    return {(k, j): M[mout[cell_index(N, k, j)]] for j in range(N) for k in range(j + 1, N + 1)}


def test_sls_schedule_reproduces_golden():
    g = load_golden("sls")
    N, n, m = 40, 4, 2
    costs = osls.assemble_costs(None, g["C"], g["D"], g["CN"], osls.Weights.identity(n, m))
    phix = emulate(g["A"], g["B"], g["E"], costs)
    gold = g["r1_phix"]
    assert max(np.abs(phix[(k, j)] - gold[k, j]).max() for (k, j) in phix) <= 1e-12


@pytest.mark.parametrize("N", [1, 2, 3, 7, 25])
def test_sls_schedule_vs_sequential(N):
    rng = np.random.default_rng(N)
    n, m = 3, 2
    A = rng.standard_normal((N, n, n)) * 0.4
    B = rng.standard_normal((N, n, m))
    E = rng.standard_normal((N, n, n)) * 0.1
    costs = osls.assemble_costs(None, rng.standard_normal((N, 2, n)), rng.standard_normal((N, 2, m)),
                                rng.standard_normal((1, n)), osls.Weights.identity(n, m))
    phix = emulate(A, B, E, costs)
    seq = osls.fastsls_sequential(A, B, E, costs)
    for (k, j), v in phix.items():
        assert np.abs(v - seq.phi_x(k, j)).max() <= 1e-9


def test_cell_layout_roundtrip():
    N = 6
    rag = [np.arange((N - j) * 2).reshape(N - j, 2) + 100 * j for j in range(N)]
    cells = ragged_to_cells(rag, N, (2,))
    back = cells_to_ragged(cells, N, 1, N + 1)
    for a, b in zip(rag, back):
        assert (a == b).all()
    assert nat.load(False).gsls_sls_ncell(N) == N * (N + 1) // 2
