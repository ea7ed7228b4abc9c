"""GPU parity: lqr.* and admm.solve_qp through the C ABI vs the CPU oracle.

Tolerances (north star): trajectories / gains within 1e-4 relative
(reference.relative_error: max|a-e| / max(1, max|e|)) in fp32 against the
fp64 oracle; ADMM iteration count and active set exactly.
"""

import numpy as np
import pytest

import oracle
from oracle import admm as oadmm, lqr as olqr
from conftest import load_golden
import problems as P

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def gs():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_07644_b200 import admm, lqr
    return lqr, admm


def rel(a, b):
    return oracle.relative_error(a, b)


def active(z, f, fp32):
    return z >= f - 1e-12


@pytest.mark.parametrize("tag", ["r6", "r5", "r12", "r61"])
def test_lqr_solve_vs_golden(gs, tag):
    lqr, _ = gs
    g = load_golden("lqr")
    nx, nu, N, seed = (int(v) for v in g[f"{tag}_dims"])
    qp = P.random_ltv_qp(np.random.default_rng(seed), nx, nu, N)
    sol = lqr.solve(qp)
    for fld in ("dx", "du", "K", "k", "p"):
        assert rel(getattr(sol, fld), g[f"{tag}_{fld}"]) <= TOL, fld
    assert rel(sol.P[0], g[f"{tag}_P0"]) <= TOL
    assert sol.scan_layers == int(g[f"{tag}_layers"])
    assert sol.dynamics_residual(qp) <= 1e-4


def test_lqr_matches_riccati_oracle(gs):
    lqr, _ = gs
    qp = P.random_ltv_qp(np.random.default_rng(0), 6, 3, 64)
    sol, ref = lqr.solve(qp), olqr.riccati(qp)
    for fld in ("dx", "du", "K"):
        assert rel(getattr(sol, fld), getattr(ref, fld)) <= TOL


@pytest.mark.parametrize("nx", [63, 65, 66, 67, 68, 76, 80])
def test_lqr_combine_sizes_64_to_80(gs, nx):
    """The k_cvf_combine<80> Gauss-Jordan column tiles (gj.cuh, NP = 80: 5 columns per
    row thread) at the state sizes where lds_of(n) and the tile width disagree, and the
    64-wide kernel's upper edge, against the float64 scan oracle."""
    lqr, _ = gs
    qp = P.random_ltv_qp(np.random.default_rng(nx), nx, 7, 9)
    sol, ref = lqr.solve(qp), olqr.solve(qp)
    for fld in ("dx", "du", "K", "k"):
        assert rel(getattr(sol, fld), getattr(ref, fld)) <= TOL, fld


def test_lqr_scalar_analytic_and_terminal_only(gs):
    lqr, _ = gs
    sol = lqr.solve(P.scalar_qp())
    assert abs(sol.du[0, 0] + 0.5) <= 1e-6 and abs(sol.dx[1, 0] - 0.5) <= 1e-6
    qp = olqr.QP(A=np.zeros((0, 2, 2)), B=np.zeros((0, 2, 1)), b=np.zeros((0, 2)), Q=np.zeros((0, 2, 2)),
                 R=np.zeros((0, 1, 1)), S=np.zeros((0, 1, 2)), q=np.zeros((0, 2)), r=np.zeros((0, 1)),
                 QN=np.eye(2), qN=np.zeros(2), C=np.zeros((0, 0, 2)), D=np.zeros((0, 0, 1)), f=np.zeros((0, 0)),
                 CN=np.zeros((0, 2)), fN=np.zeros(0), dx0=np.array([1.0, 2.0]))
    sol = lqr.solve(qp)
    assert (sol.dx == np.array([[1.0, 2.0]])).all() and sol.du.shape[0] == 0


def test_lqr_feedback_law_and_layers(gs):
    lqr, _ = gs
    rng = np.random.default_rng(3)
    for N in (1, 5, 33, 100):
        qp = P.random_ltv_qp(rng, 3, 2, N)
        sol = lqr.solve(qp)
        ref = olqr.solve(qp)
        assert sol.scan_layers == ref.scan_layers
        assert rel(sol.dx, ref.dx) <= TOL


def test_cache_bitwise_and_perturbed(gs):
    lqr, _ = gs
    g = load_golden("lqr")
    qp = P.random_ltv_qp(np.random.default_rng(1), 5, 2, 29)
    sol, cache = lqr.build_cache(qp, generation=4)
    again = lqr.solve_cached(lqr.LqrLinearTerms(qp.q, qp.r, qp.qN), cache, 4)
    for fld in ("dx", "du", "K", "k", "P", "p"):
        assert (np.asarray(getattr(sol, fld)) == np.asarray(getattr(again, fld))).all(), fld
    _, cache0 = lqr.build_cache(qp, generation=0)
    fast = lqr.solve_cached(lqr.LqrLinearTerms(g["pert_q"], g["pert_r"], g["pert_qN"]), cache0, 0)
    for fld in ("dx", "du", "k", "p"):
        assert rel(getattr(fast, fld), g[f"pert_{fld}"]) <= TOL
    full = lqr.solve(qp.replace(q=g["pert_q"], r=g["pert_r"], qN=g["pert_qN"]))
    for fld in ("dx", "du", "k", "p"):
        assert (getattr(full, fld) == getattr(fast, fld)).all(), fld
    with pytest.raises(lqr.CacheInvalidatedError, match="cache invalidated"):
        lqr.solve_cached(lqr.LqrLinearTerms(qp.q, qp.r, qp.qN), cache0, 1)


def test_lqr_errors(gs):
    lqr, _ = gs
    with pytest.raises(lqr.SingularStageError, match="stage 0"):
        lqr.solve(P.scalar_qp(R=np.full((1, 1, 1), -1.0)))
    # P C = -I makes I + P C singular: left (P=0,C=1), right (P=-1,C=0) -> QN = -1 terminal, C0 = 1
    qp = P.scalar_qp(Q=np.zeros((1, 1, 1)), QN=-np.ones((1, 1)), R=np.ones((1, 1, 1)), B=np.ones((1, 1, 1)))
    with pytest.raises(lqr.IllConditionedCombineError, match="ill-conditioned combine"):
        lqr.solve(qp)


# --- ADMM ------------------------------------------------------------------------

SET_A = dict(rho0=0.1, sigma=10, tol_primal=1e-4, tol_dual=1e-4, max_iter=4000)


def test_admm_double_integrator_golden(gs):
    _, admm = gs
    g = load_golden("admm")
    qp = P.double_integrator()
    res = admm.solve_qp(qp, admm.AdmmSettings(**SET_A))
    assert res.stats.iterations == int(g["di_iters"]) == 109
    assert res.stats.cache_builds == int(g["di_builds"])
    assert res.stats.rho_changes == int(g["di_rho_changes"])
    f = oadmm.offsets(qp)
    assert (active(res.state.z, f, True) == g["di_active"]).all()
    assert rel(res.dx, g["di_dx"]) <= TOL and rel(res.du, g["di_du"]) <= TOL
    assert rel(res.state.lam, g["di_lam"]) <= TOL


def test_admm_seeded_batch_golden(gs):
    _, admm = gs
    g = load_golden("admm")
    f = oadmm.offsets(P.double_integrator())
    for i, x0 in enumerate(g["dib_x0"]):
        res = admm.solve_qp(P.double_integrator(dx0=x0), admm.AdmmSettings(**SET_A))
        assert res.stats.iterations == int(g["dib_iters"][i]), i
        assert (active(res.state.z, f, True) == g["dib_active"][i]).all()
        assert rel(res.dx, g["dib_dx"][i]) <= TOL


@pytest.mark.parametrize("i", [0, 1, 2])
def test_admm_random_golden(gs, i):
    """The reference's random fixtures (test_admm.py:118-129) at tol 1e-6: iteration count
    (127 / 70 / 82), rho changes and active set exactly, solution within 1e-4."""
    _, admm = gs
    g = load_golden("admm")
    qp = olqr.QP(**{k: g[f"rnd{i}_qp_{k}"] for k in olqr.FIELDS})
    res = admm.solve_qp(qp, admm.AdmmSettings(tol_primal=1e-6, tol_dual=1e-6))
    assert res.stats.converged
    assert res.stats.iterations == int(g[f"rnd{i}_iters"])
    assert res.stats.rho_changes == int(g[f"rnd{i}_rho_changes"])
    ref = oadmm.solve_qp(qp, oadmm.Settings(tol_primal=1e-6, tol_dual=1e-6))
    f = oadmm.offsets(qp)
    assert (active(res.state.z, f, True) == active(ref.state.z, f, False)).all()
    assert rel(res.dx, g[f"rnd{i}_dx"]) <= TOL and rel(res.du, g[f"rnd{i}_du"]) <= TOL
    assert rel(res.state.lam, g[f"rnd{i}_lam"]) <= TOL
    obj = P.qp_objective(qp, res.dx, res.du)
    assert abs(obj - float(g[f"rnd{i}_obj"])) <= 1e-4 * max(1.0, abs(float(g[f"rnd{i}_obj"])))


def test_admm_no_inequalities_single_iteration(gs):
    lqr, admm = gs
    qp = P.scalar_qp()
    res = admm.solve_qp(qp, admm.AdmmSettings(tol_primal=1e-9, tol_dual=1e-9))
    plain = lqr.solve(qp)
    assert res.stats.iterations == 1
    assert (res.du == plain.du).all() and (res.dx == plain.dx).all()


def test_admm_scalar_active_constraint(gs):
    _, admm = gs
    qp = P.scalar_qp(Q=np.zeros((1, 1, 1)), C=np.zeros((1, 1, 1)), D=np.array([[[-1.0]]]), f=np.zeros((1, 1)))
    res = admm.solve_qp(qp, admm.AdmmSettings(tol_primal=1e-6, tol_dual=1e-6))
    assert res.stats.converged
    assert abs(res.du[0, 0]) <= 1e-5 and abs(res.dx[1, 0] - 1.0) <= 1e-5
    lam, _ = res.stage_duals(qp)
    assert abs(lam[0, 0] - 1.0) <= 1e-4


def test_admm_warm_start_mutated_and_max_iter(gs):
    _, admm = gs
    rng = np.random.default_rng(0)
    qp = P.random_ltv_qp(rng, 3, 2, 10, nc=2)
    st = admm.AdmmSettings(tol_primal=1e-5, tol_dual=1e-5)
    first = admm.solve_qp(qp, st)
    assert first.stats.converged
    warm = first.state
    again = admm.solve_qp(qp, st, warm_start=warm)
    assert again.state is warm
    assert again.stats.converged and again.stats.iterations <= 2
    qp = P.random_ltv_qp(rng, 3, 2, 10, nc=3)
    res = admm.solve_qp(qp, admm.AdmmSettings(tol_primal=1e-12, tol_dual=1e-12, max_iter=5))
    assert not res.stats.converged and res.stats.iterations == 5


def test_admm_matches_oracle_trace_random(gs):
    """Iteration count and active set vs the oracle on structured random QPs."""
    _, admm = gs
    for seed in range(4):
        rng = np.random.default_rng(100 + seed)
        qp = P.random_ltv_qp(rng, 8, 3, 30, nc=0)
        # box on inputs (well-conditioned ADMM)
        D = np.tile(np.vstack([np.eye(3), -np.eye(3)]), (30, 1, 1))
        qp = qp.replace(C=np.zeros((30, 6, 8)), D=D, f=np.full((30, 6), 0.3))
        s = dict(rho0=0.1, sigma=10, tol_primal=1e-4, tol_dual=1e-4, max_iter=2000)
        res = admm.solve_qp(qp, admm.AdmmSettings(**s))
        ref = oadmm.solve_qp(qp, oadmm.Settings(**s))
        assert res.stats.iterations == ref.stats.iterations, seed
        f = oadmm.offsets(qp)
        assert (active(res.state.z, f, True) == active(ref.state.z, f, False)).all()
        assert rel(res.du, ref.du) <= TOL
