"""Numerics of the factored (Woodbury) CVF combine in float32 vs the dense float32 combine.

The CVF combine (lqr.py:226-239) inverts M1 = I + P_r C_l.  Every leaf's C is
B R^-1 B' (rank m), and a combine's C = Psi C_l A_r' + C_r has rank <= rank C_l +
rank C_r.  Carrying C = F F' (F: n x r) gives, with S = I_r + F' P_r F = L L',
Fh = F L^-T, V = P_r Fh:

    M1^-1 P_r = P_r - V V'        P = A_l' (P_r - V V') A_l + P_l
    A = A_r A_l - (A_r Fh)(V' A_l) C = (A_r Fh)(A_r Fh)' + C_r  -> factor [A_r Fh, F_r]

This probe runs the SLS reverse grid scan (sls.py:227-280) of one cfg-D / E-RTI
scenario per column with the reference's tree, in float32, both ways, and reports
the relative error of the scan outputs P against the float64 oracle.

    python tools/probe/lowrank_numerics.py [q61|h75] [rmax]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from oracle import tree  # noqa: E402

f32 = np.float32


class El:
    __slots__ = ("P", "A", "F", "C")

    def __init__(self, P, A, F=None, C=None):
        self.P, self.A, self.F, self.C = P, A, F, C


def dense_combine(l, r):
    n = l.P.shape[0]
    I = np.eye(n, dtype=f32)
    Cl = l.C if l.C is not None else l.F @ l.F.T
    Cr = r.C if r.C is not None else r.F @ r.F.T
    Minv = np.linalg.inv(I + r.P @ Cl).astype(f32)
    M2inv = np.linalg.inv(I + Cl @ r.P).astype(f32)
    P = l.A.T @ (Minv @ r.P) @ l.A + l.P
    A = r.A @ M2inv @ l.A
    C = r.A @ M2inv @ Cl @ r.A.T + Cr
    return El(P.astype(f32), A.astype(f32), None, C.astype(f32))


def lowrank_combine(l, r, rmax):
    if l.F is None:
        return dense_combine(l, r)
    F = l.F
    n, k = F.shape
    if k == 0:
        P = l.A.T @ r.P @ l.A + l.P
        return El(P, r.A @ l.A, r.F, r.C)
    W = r.P @ F
    S = np.eye(k, dtype=f32) + F.T @ W
    L = np.linalg.cholesky(S).astype(f32)
    Li = np.linalg.inv(L).astype(f32)
    Fh = F @ Li.T
    V = W @ Li.T
    Pm = r.P - V @ V.T
    P = l.A.T @ Pm @ l.A + l.P
    U = r.A @ Fh
    A = r.A @ l.A - U @ (V.T @ l.A)
    if r.F is not None and U.shape[1] + r.F.shape[1] <= rmax:
        return El(P.astype(f32), A.astype(f32), np.concatenate([U, r.F], axis=1).astype(f32), None)
    Cr = r.C if r.C is not None else r.F @ r.F.T
    return El(P.astype(f32), A.astype(f32), None, (U @ U.T + Cr).astype(f32))


def grid_scan(Pel, Ael, Fel, Cel, combine):
    """Per column j: the reverse scan of positions 0..N (terminal at N)."""
    def op(lhs, rhs):
        a, b = lhs[0], rhs[0]
        out = np.empty(len(a), dtype=object)
        for i in range(len(a)):
            out[i] = combine(a[i], b[i])
        return (out,), ()
    L = len(Pel)
    items = np.empty(L, dtype=object)
    for i in range(L):
        items[i] = El(Pel[i], Ael[i], Fel[i], Cel[i])
    n = Pel[0].shape[0]
    unit = El(np.zeros((n, n), f32), np.eye(n, dtype=f32), np.zeros((n, 0), f32), None)

    def mk(k):
        arr = np.empty(k, dtype=object)
        for i in range(k):
            arr[i] = unit
        return (arr,)
    out, _ = tree.scan((items,), op, mk, reverse=True)
    return [e.P for e in out[0]]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "q61"
    rmax = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    from paper_2604_07644_b200 import scenarios as S
    wl = S.rti_workload(tag)
    m = wl.model
    x = wl.scenario_states(5, 1)[0]
    prev = oracle.sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    qp = oracle.sqp.linearize(m, prev, None, x)
    du = oracle.sls.Duals.zero(wl.N, m.nc, m.nf, S.EPS)
    du.tau, du.tau_term = wl.tau, wl.tau_term
    w = oracle.sls.Weights(np.eye(m.nx), S.RBAR * np.eye(m.nu), np.eye(m.nx))
    costs = oracle.sls.assemble_costs(du, qp.C, qp.D, qp.CN, w)
    N, n = wl.N, m.nx
    A, B = qp.A, qp.B
    worst = {"dense": 0.0, "lowrank": 0.0}
    for j in range(0, N - 1, 4):
        Pel, Ael, Fel, Cel = [], [], [], []
        Pref, Aref, Cref = [], [], []
        for k in range(j + 1, N):
            Qx, Qu, Qux = costs.Qx[j][k - j - 1], costs.Qu[j][k - j - 1], costs.Qux[j][k - j - 1]
            Lq = np.linalg.cholesky(Qu)
            Qi = np.linalg.inv(Qu)
            P = Qx - Qux.T @ Qi @ Qux
            Aa = A[k] - B[k] @ Qi @ Qux
            F = B[k] @ np.linalg.inv(Lq).T
            Pel.append(P.astype(f32)); Ael.append(Aa.astype(f32)); Fel.append(F.astype(f32)); Cel.append(None)
            Pref.append(P); Aref.append(Aa); Cref.append(B[k] @ Qi @ B[k].T)
        Pel.append(costs.Qx_term[j].astype(f32)); Ael.append(np.zeros((n, n), f32))
        Fel.append(np.zeros((n, 0), f32)); Cel.append(None)
        Pref.append(costs.Qx_term[j]); Aref.append(np.zeros((n, n))); Cref.append(np.zeros((n, n)))
        out64, _ = tree.scan((np.array(Pref), np.array(Aref), np.array(Cref)),
                             lambda l, r: ((lambda t: (t[0], t[1], t[2]))(oracle.lqr.cvf_matrix(l[0], l[1], l[2], r[0], r[1], r[2])), ()),
                             lambda c: (np.zeros((c, n, n)), np.tile(np.eye(n), (c, 1, 1)), np.zeros((c, n, n))),
                             reverse=True)
        ref = out64[0]
        Pd = grid_scan(Pel, Ael, [None] * len(Pel), [F @ F.T if F.shape[1] else np.zeros((n, n), f32) for F in Fel],
                       dense_combine)
        Pl = grid_scan(Pel, Ael, Fel, Cel, lambda l, r: lowrank_combine(l, r, rmax))
        ed = max(oracle.relative_error(Pd[i], ref[i]) for i in range(len(ref)))
        el = max(oracle.relative_error(Pl[i], ref[i]) for i in range(len(ref)))
        worst["dense"] = max(worst["dense"], ed)
        worst["lowrank"] = max(worst["lowrank"], el)
        print(f"column {j:2d}: dense f32 {ed:.2e}  lowrank f32 {el:.2e}  (max |P| {np.abs(ref).max():.3g})")
    print(tag, "worst", worst)


if __name__ == "__main__":
    main()
