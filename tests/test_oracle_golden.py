"""Pin the CPU oracle against outputs of the real reference (tests/golden/*.npz).

CPU-only.  These tests are what make the oracle trustworthy as the checker
for the CUDA path: every fixture was produced by /root/reference's scanmpc
(see tests/golden/make_golden.py), and the oracle must reproduce it to
float64 rounding (1e-9 relative), discrete outcomes exactly.
"""

import os

import numpy as np
import pytest

import oracle
from oracle import admm as oadmm, lqr as olqr, sls as osls, sqp as osqp, tree
from conftest import GOLDEN, load_golden
import problems as P
from paper_2604_07644_b200 import models as M

TOL = 1e-9


def rel(a, b):
    return oracle.relative_error(a, b)


def qp_from(g, prefix):
    return olqr.QP(**{k: g[prefix + k] for k in olqr.FIELDS})


# --- scan -------------------------------------------------------------------------

def test_scan_golden():
    g = load_golden("scan")
    ints = g["ints"].tolist()
    assert tree.scan_list(ints, lambda a, b: a + b, 0) == g["fwd"].tolist()
    assert tree.scan_list(ints, lambda a, b: a + b, 0, reverse=True) == g["rev"].tolist()
    suf = tree.scan_list(list(g["mats"]), lambda a, b: a @ b, np.eye(2), reverse=True)
    assert np.abs(np.array(suf) - g["suffix"]).max() <= 1e-12
    for L, d in g["depths"]:
        assert tree.depth(int(L)) == d


@pytest.mark.parametrize("length", [1, 2, 3, 8, 17, 1000])
def test_scan_layer_count(length):
    t = tree.Tally()
    tree.scan_list(list(range(length)), lambda a, b: a + b, 0, tally=t)
    assert t.layers == tree.depth(length)


def test_scan_empty_rejected():
    with pytest.raises(ValueError, match="empty scan"):
        tree.scan_list([], lambda a, b: a + b, 0)


# --- LQR --------------------------------------------------------------------------

@pytest.mark.parametrize("tag", ["r6", "r5", "r12", "r61"])
def test_lqr_golden(tag):
    g = load_golden("lqr")
    nx, nu, N, seed = (int(v) for v in g[f"{tag}_dims"])
    qp = P.random_ltv_qp(np.random.default_rng(seed), nx, nu, N)
    chk = sum(float(np.abs(getattr(qp, k)).sum()) for k in olqr.FIELDS)
    assert chk == pytest.approx(float(g[f"{tag}_checksum"]), rel=1e-12)
    sol = olqr.solve(qp)
    for fld in ("dx", "du", "K", "k", "p"):
        assert rel(getattr(sol, fld), g[f"{tag}_{fld}"]) <= TOL, fld
    assert rel(sol.P[0], g[f"{tag}_P0"]) <= TOL
    assert sol.scan_layers == int(g[f"{tag}_layers"])


def test_lqr_cached_golden():
    g = load_golden("lqr")
    qp = P.random_ltv_qp(np.random.default_rng(1), 5, 2, 29)
    _, cache = olqr.build_cache(qp, generation=0)
    fast = olqr.solve_cached(g["pert_q"], g["pert_r"], g["pert_qN"], cache, 0)
    for fld in ("dx", "du", "k", "p"):
        assert rel(getattr(fast, fld), g[f"pert_{fld}"]) <= TOL
    full = olqr.solve(qp.replace(q=g["pert_q"], r=g["pert_r"], qN=g["pert_qN"]))
    for fld in ("dx", "du", "K", "k", "P", "p"):
        assert (getattr(full, fld) == getattr(fast, fld)).all()
    with pytest.raises(olqr.CacheInvalidatedError, match="cache invalidated"):
        olqr.solve_cached(qp.q, qp.r, qp.qN, cache, 1)


def test_lqr_scalar_and_riccati():
    g = load_golden("lqr")
    s = olqr.solve(P.scalar_qp())
    assert abs(s.du[0, 0] + 0.5) <= 1e-12 and abs(s.dx[1, 0] - 0.5) <= 1e-12
    assert (s.du == g["scalar_du"]).all()
    qp = P.random_ltv_qp(np.random.default_rng(0), 6, 3, 64)
    a, b = olqr.solve(qp), olqr.riccati(qp)
    for fld in ("dx", "du", "K"):
        assert rel(getattr(a, fld), getattr(b, fld)) <= 1e-8


def test_lqr_errors():
    with pytest.raises(olqr.SingularStageError, match="stage 0"):
        olqr.leaves(P.scalar_qp(R=np.full((1, 1, 1), -1.0)))
    one = lambda v: np.full((1, 1, 1), v)  # noqa: E731
    lhs = (one(0.0), np.zeros((1, 1)), one(1.0), one(1.0), np.zeros((1, 1)))
    rhs = (one(-1.0), np.zeros((1, 1)), one(1.0), one(0.0), np.zeros((1, 1)))
    with pytest.raises(olqr.IllConditionedCombineError, match="ill-conditioned combine"):
        olqr.cvf_op(lhs, rhs)


# --- ADMM -------------------------------------------------------------------------

SET_A = oadmm.Settings(rho0=0.1, sigma=10, tol_primal=1e-4, tol_dual=1e-4, max_iter=4000)


def test_admm_double_integrator_golden():
    g = load_golden("admm")
    qp = qp_from(g, "di_qp_")
    res = oadmm.solve_qp(qp, SET_A)
    assert res.stats.iterations == int(g["di_iters"]) == 109
    assert res.stats.rho_changes == int(g["di_rho_changes"])
    assert res.stats.cache_builds == int(g["di_builds"]) == 2
    f = oadmm.offsets(qp)
    act = res.state.z >= f - 1e-12
    assert (act == g["di_active"]).all() and act.sum() == 45
    assert rel(res.dx, g["di_dx"]) <= 1e-8 and rel(res.du, g["di_du"]) <= 1e-8
    assert rel(res.state.lam, g["di_lam"]) <= 1e-8


def test_admm_batch_golden():
    g = load_golden("admm")
    for i, x0 in enumerate(g["dib_x0"][:3]):
        res = oadmm.solve_qp(P.double_integrator(dx0=x0), SET_A)
        assert res.stats.iterations == int(g["dib_iters"][i])
        assert rel(res.dx, g["dib_dx"][i]) <= 1e-7


@pytest.mark.parametrize("i", [0, 1, 2])
def test_admm_random_golden(i):
    g = load_golden("admm")
    qp = qp_from(g, f"rnd{i}_qp_")
    res = oadmm.solve_qp(qp, oadmm.Settings(tol_primal=1e-6, tol_dual=1e-6))
    assert res.stats.iterations == int(g[f"rnd{i}_iters"])
    assert rel(res.dx, g[f"rnd{i}_dx"]) <= 1e-8
    obj = P.qp_objective(qp, res.dx, res.du)
    assert abs(obj - float(g[f"rnd{i}_obj"])) <= 1e-4 * max(1.0, abs(float(g[f"rnd{i}_obj"])))


def test_admm_settings_and_rho_rules():
    with pytest.raises(ValueError, match="sigma"):
        oadmm.Settings(sigma=1)
    st = oadmm.State.fresh(2, 1.0)
    st.lam = np.array([2.0, -1.0])
    out = oadmm.update_rho(st, 100.0, 1.0, oadmm.Settings())
    assert out.rho == pytest.approx(10.0) and out.generation == 1
    st = oadmm.State.fresh(1, 1.0)
    assert oadmm.update_rho(st, 4.0, 1.0, oadmm.Settings()).generation == 0


# --- SLS --------------------------------------------------------------------------

def _resp_from(g, prefix, N):
    return osls.Response(P.unpack_lower(g[prefix + "phix"], N, 1, N + 1),
                         P.unpack_lower(g[prefix + "phiu"], N, 1, N),
                         P.unpack_lower(g[prefix + "gain"], N, 1, N), N, 4, 2)


def test_sls_golden():
    g = load_golden("sls")
    N, nx, nu = 40, 4, 2
    w = osls.Weights.identity(nx, nu)
    costs = osls.assemble_costs(None, g["C"], g["D"], g["CN"], w)
    resp = osls.synthesize(g["A"], g["B"], g["E"], costs)
    ref = _resp_from(g, "r1_", N)
    for j in range(N):
        assert rel(resp.Phi_x[j], ref.Phi_x[j]) <= TOL
        assert rel(resp.Phi_u[j], ref.Phi_u[j]) <= TOL
        assert rel(resp.gains[j], ref.gains[j]) <= TOL
    t = osls.tighten(resp, g["C"], g["D"], g["CN"])
    assert rel(t.h, g["h"]) <= TOL and rel(t.hf, g["hf"]) <= TOL
    du = osls.compute_duals(g["lam_s"], g["lam_t"], resp, g["C"], g["D"], g["CN"], 1e-6)
    assert rel(P.pack_lower(du.tau, N, 1, N, (2,)), g["tau"]) <= TOL
    assert rel(du.tau_term, g["tau_term"]) <= TOL
    w2 = osls.Weights(2 * np.eye(nx), 3 * np.eye(nu), np.eye(nx))
    resp2 = osls.synthesize(g["A"], g["B"], g["E"], osls.assemble_costs(du, g["C"], g["D"], g["CN"], w2))
    t2 = osls.tighten(resp2, g["C"], g["D"], g["CN"])
    assert rel(t2.h, g["h2"]) <= TOL and rel(t2.hf, g["hf2"]) <= TOL
    assert osls.sls_cost(resp2, w2) == pytest.approx(float(g["cost2"]), rel=1e-10)
    seq = osls.fastsls_sequential(g["A"], g["B"], g["E"], costs)
    assert max(rel(seq.Phi_x[j], resp.Phi_x[j]) for j in range(N)) <= 1e-8


def test_sls_hand_two_stage():
    """test_reference.py:86-98: K = -1/2, Phi^x_{2,0} = 1/2, Phi^u_{1,0} = -1/2."""
    costs = osls.Costs([np.ones((1, 1, 1)), np.zeros((0, 1, 1))], [np.ones((1, 1, 1)), np.zeros((0, 1, 1))],
                       [np.zeros((1, 1, 1)), np.zeros((0, 1, 1))], np.ones((2, 1, 1)))
    ones = np.ones((2, 1, 1))
    for fn in (osls.fastsls_sequential, osls.synthesize):
        r = fn(ones, ones, ones, costs)
        assert r.gains[0][0, 0, 0] == pytest.approx(-0.5)
        assert r.phi_x(2, 0)[0, 0] == pytest.approx(0.5)
        assert r.phi_u(1, 0)[0, 0] == pytest.approx(-0.5)


# --- models (our host plants vs the reference's) ---------------------------------

@pytest.mark.parametrize("tag,model", [
    ("dubins", M.DubinsCar(obstacles=((1.0, 0.5, 0.3),))),
    ("quad", M.PlanarQuadrotor(obstacles=((1.5, 0.0, 0.35),))),
    ("pend2", M.NLinkPendulum(n_links=2)),
    ("pend4", M.NLinkPendulum(n_links=4, e_rate=0.05)),
])
def test_models_golden(tag, model):
    g = load_golden("models")
    for i, (x, u) in enumerate(zip(g[f"{tag}_x"], g[f"{tag}_u"])):
        assert np.abs(model.step(x, u) - g[f"{tag}_step"][i]).max() <= 1e-12
        A, B = model.jacobians(x, u)
        assert np.abs(A - g[f"{tag}_A"][i]).max() <= 1e-10
        assert np.abs(B - g[f"{tag}_B"][i]).max() <= 1e-10
        assert np.abs(model.stage_constraints(x, u) - g[f"{tag}_g"][i]).max() <= 1e-12
        C, D = model.stage_constraint_jacobians(x, u)
        assert np.abs(C - g[f"{tag}_C"][i]).max() <= 1e-12 and (D == g[f"{tag}_D"][i]).all()
        assert (model.disturbance(x) == g[f"{tag}_E"][i]).all()
        assert np.abs(model.terminal_constraints(x) - g[f"{tag}_gf"][i]).max(initial=0) <= 1e-12


# --- RTI robust step --------------------------------------------------------------

def rti_case(tag):
    """(model, settings) for a golden RTI case; mirrors make_golden.gen_rti."""
    if tag == "pq":
        model = M.PlanarQuadrotor(dt=0.05, thrust_max=30.0, goal=(2.6, 0, 0, 0, 0, 0), obstacles=((1.5, 0.0, 0.35),))
        st = osqp.Settings(max_sqp_iters=30, kkt_tol=2e-3,
                           admm=oadmm.Settings(rho0=10.0, tol_primal=1e-3, tol_dual=1e-3, max_iter=3000))
        Q = np.diag([20.0, 20, 1, 4, 4, 0.5])
        rs = osls.RobustSettings(sqp=st, weights=osls.Weights(Q, 0.3 * np.eye(2), Q), eps=1e-4)
    else:
        model = M.quadruped61() if tag == "q61" else M.humanoid75()
        st = osqp.Settings(max_sqp_iters=30, kkt_tol=1e-3,
                           admm=oadmm.Settings(rho0=1.0, tol_primal=1e-3, tol_dual=1e-3, max_iter=500))
        rs = osls.RobustSettings(sqp=st, eps=1e-4,
                                 weights=osls.Weights(np.eye(model.nx), 10 * np.eye(model.nu), np.eye(model.nx)))
    return model, rs


def rti_inputs(g, tag, model):
    prev = osqp.Trajectory(g[f"{tag}_prev_x"], g[f"{tag}_prev_u"], float(g[f"{tag}_prev_dt"]))
    N = prev.N
    tau = None
    if g[f"{tag}_tau_in"].size:
        tau = osls.Duals.zero(N, model.nc, model.nf, 1e-4)
        tau.tau = P.unpack_lower(g[f"{tag}_tau_in"], N, 1, N)
        tau.tau_term = g[f"{tag}_tau_term_in"]
    return g[f"{tag}_xbar0"], prev, tau


@pytest.mark.parametrize("tag", ["pq", "q61"])
def test_rti_robust_golden(tag):
    if not os.path.exists(os.path.join(GOLDEN, "rti.npz")):
        pytest.skip("rti golden not generated")
    g = load_golden("rti")
    model, rs = rti_case(tag)
    x, prev, tau = rti_inputs(g, tag, model)
    r = osls.rti_robust_step(model, x, prev, tau, rs)
    assert r.stats.admm_iterations == int(g[f"{tag}_admm_iters"])
    assert rel(r.u0, g[f"{tag}_u0"]) <= 1e-7
    assert rel(r.tightening.h, g[f"{tag}_h"]) <= 1e-7
    assert rel(r.plan.x, g[f"{tag}_plan_x"]) <= 1e-7
    assert rel(P.pack_lower(r.tau.tau, prev.N, 1, prev.N, (model.nc,)), g[f"{tag}_tau_out"]) <= 1e-6


# --- rollout (rollout.py:41-180) ----------------------------------------------------

@pytest.mark.parametrize("tag", P.ROLLOUT_TAGS)
def test_rollout_golden(tag):
    from oracle import rollout as orl
    g = load_golden("rollout")
    mdl = P.rollout_model(tag)
    x, u, N = g[f"{tag}_x"], g[f"{tag}_u"], int(g[f"{tag}_N"])
    phiu = g[f"{tag}_phiu"]
    h = g[f"{tag}_h"]
    # samplers reproduce the reference's seeded streams bit for bit
    nx = mdl.nx
    assert np.array_equal(orl.sample_disturbance("uniform_ball", nx, N, 11), g[f"{tag}_dist"][0])
    assert np.array_equal(orl.sample_disturbance("boundary", nx, N, 12), g[f"{tag}_dist"][1])
    rows = orl.adversarial_rows(mdl, x, u)
    assert rel(rows, g[f"{tag}_rows"]) <= TOL
    assert np.array_equal(orl.sample_disturbance("adversarial", nx, N, 0, rows=g[f"{tag}_rows"]), g[f"{tag}_dist"][2])
    for i, d in enumerate(g[f"{tag}_dist"]):
        r = orl.closed_loop(mdl, x, u, lambda k, j: phiu[k, j], d, h)
        for f in ("x", "u", "w", "stage_g", "terminal_g"):
            assert rel(getattr(r, f), g[f"{tag}_rec_{f}"][i]) <= TOL, (tag, i, f)
        tm, gtm = r.tube_margin, g[f"{tag}_rec_tube_margin"][i]
        assert np.array_equal(np.isinf(tm), np.isinf(gtm))
        assert rel(np.where(np.isinf(tm), 0, tm), np.where(np.isinf(gtm), 0, gtm)) <= TOL
        assert r.safe == bool(g[f"{tag}_rec_safe"][i])
        assert r.tube_ok == bool(g[f"{tag}_rec_tube_ok"][i])
        assert r.disturbance_model_violated == bool(g[f"{tag}_rec_disturbance_model_violated"][i])
        assert abs(r.max_w_norm - g[f"{tag}_rec_max_w_norm"][i]) <= TOL * max(1, r.max_w_norm)
    r = orl.closed_loop(mdl, x, u, lambda k, j: phiu[k, j], g[f"{tag}_dist"][0], None)
    assert np.isinf(r.tube_margin).all() and r.tube_ok == bool(g[f"{tag}_nt_tube_ok"])
    rec0 = orl.closed_loop(mdl, x, u, lambda k, j: phiu[k, j], g[f"{tag}_dist"][0], h)
    sup = orl.superposition_check(x, lambda k, j: g[f"{tag}_phix"][k, j], rec0.w, rec0.x)
    assert abs(sup - float(g[f"{tag}_superposition"])) <= 1e-9 * max(1.0, sup)


def test_rollout_sampler_errors():
    from oracle import rollout as orl
    with pytest.raises(ValueError, match="adversarial sampling needs"):
        orl.sample_disturbance("adversarial", 3, 4, 0)
    with pytest.raises(ValueError, match="unknown disturbance kind"):
        orl.sample_disturbance("gaussian", 3, 4, 0)
    with pytest.raises(ValueError, match="rows must be"):
        orl.sample_disturbance("adversarial", 3, 4, 0, rows=np.ones((3, 3)))


# --- benched batch, nominal RTI, configs B / C / E, error paths (make_golden.py) -------------

def _oracle_rti(tag, idx, robust=True):
    from paper_2604_07644_b200 import scenarios as S
    import bench
    wl = S.rti_workload(tag)
    m = wl.model
    rs = bench.oracle_settings(m)
    x = wl.scenario_states(idx, 1)[0]
    prev = osqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    st = oadmm.State.fresh(wl.N * m.nc + m.nf, rs.sqp.admm.rho0)
    if robust:
        tau = osls.Duals.zero(wl.N, m.nc, m.nf, rs.eps)
        tau.tau, tau.tau_term = wl.tau, wl.tau_term
        r = osls.rti_robust_step(m, x, prev, tau, rs, warm_admm=st)
        qp = osqp.linearize(m, prev, r.tightening, x)
    else:
        r = osqp.rti_step(m, x, prev, rs.sqp, warm_admm=st)
        qp = osqp.linearize(m, prev, None, x)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    return r, st, st.z >= f - 1e-12


@pytest.mark.parametrize("tag,idx", [("q61", 0), ("q61", 5), ("q61", 37), ("h75", 9)])
def test_batch_golden(tag, idx):
    """The oracle reproduces the reference on benched scenarios (bench.py's CPU arms)."""
    g = load_golden("batch")
    r, st, act = _oracle_rti(tag, idx)
    assert r.stats.admm_iterations == g[f"{tag}_iters"][idx]
    assert st.generation == g[f"{tag}_rho_changes"][idx]
    assert (act == g[f"{tag}_active"][idx]).all()
    assert rel(r.u0, g[f"{tag}_u0"][idx]) <= 1e-7
    assert rel(r.tightening.h, g[f"{tag}_h"][idx]) <= 1e-7


def test_nominal_golden():
    g = load_golden("nominal")
    r, st, act = _oracle_rti("q61", 2, robust=False)
    assert r.stats.admm_iterations == g["q61_iters"][2]
    assert (act == g["q61_active"][2]).all()
    assert rel(r.u0, g["q61_u0"][2]) <= 1e-7 and rel(r.plan.x, g["q61_plan_x"][2]) <= 1e-7


def _qp_counter(monkeypatch):
    calls = []
    orig = oadmm.solve_qp

    def wrap(*a, **k):
        r = orig(*a, **k)
        calls.append((r.stats.iterations, int(r.stats.converged), r.stats.rho_changes, r.stats.cache_builds))
        return r
    monkeypatch.setattr(osqp.admm, "solve_qp", wrap)
    return calls


def test_cfgb_golden(monkeypatch):
    from paper_2604_07644_b200 import scenarios as S
    g = load_golden("cfgb")
    calls = _qp_counter(monkeypatch)
    m = S.cfgb_model()
    x0 = S.quad12_start()
    xg, ug = S.hover_guess(m, x0, S.CFGB["N"])
    st = osqp.Settings(admm=oadmm.Settings(**S.CFGB["admm"]), **S.CFGB["sqp"])
    r = osqp.solve_nmpc(m, x0, st, osqp.Trajectory(xg, ug, m.dt))
    assert (np.array(calls) == g["qp_calls"]).all()
    assert r.stats.iterations == int(g["sqp_iters"]) and r.stats.converged
    assert rel(r.trajectory.x, g["x"]) <= 1e-7 and rel(r.lam_stage, g["lam_s"]) <= 1e-6


def test_cfgc_golden():
    """Pins the oracle's solve_robust (sls.py:400-469) against the real reference."""
    from paper_2604_07644_b200 import scenarios as S
    g = load_golden("cfgc")
    m = S.cfgc_model()
    x0 = S.quad12_start()
    N = S.CFGC["N"]
    xg, ug = S.hover_guess(m, x0, N)
    st = osqp.Settings(admm=oadmm.Settings(**S.CFGC["admm"]), **S.CFGC["sqp"])
    rs = osls.RobustSettings(sqp=st, weights=osls.Weights.identity(m.nx, m.nu), eps=S.CFGC["eps"],
                             tol_h=S.CFGC["tol_h"], max_alternations=S.CFGC["max_alternations"])
    r = osls.solve_robust(m, x0, rs, initial=osqp.Trajectory(xg, ug, m.dt))
    assert r.stats.alternations == int(g["alternations"]) and r.stats.converged == bool(g["converged"])
    assert r.stats.sqp_iterations == int(g["sqp_iters"])
    assert rel(r.trajectory.x, g["x"]) <= 1e-6 and rel(r.tightening.h, g["h"]) <= 1e-6
    assert rel(P.pack_lower(r.duals.tau, N, 1, N, (m.nc,)), g["tau"]) <= 1e-6


def test_cfge_golden():
    from paper_2604_07644_b200 import scenarios as S
    g = load_golden("cfge")
    m = S.cfge_model()
    N = S.CFGE["N"]
    x, u = S.cfge_trajectory(m, N)
    qp = osqp.linearize(m, osqp.Trajectory(x, u, m.dt), None, S.cfge_start(m))
    assert sum(float(np.abs(getattr(qp, k)).sum()) for k in olqr.FIELDS) == pytest.approx(float(g["checksum"]),
                                                                                          rel=1e-12)
    res = oadmm.solve_qp(qp, oadmm.Settings(**S.CFGE["admm"]))
    assert res.stats.iterations == int(g["iters"]) and res.stats.rho_changes == int(g["rho_changes"])
    f = oadmm.offsets(qp)
    act = res.state.z >= f - 1e-12
    assert (act == np.unpackbits(g["active"])[: f.size].astype(bool)).all()
    assert rel(res.dx, g["dx"].astype(float)) <= 1e-6


def test_error_goldens():
    g = load_golden("errors")
    qp = olqr.QP(**{k: g[f"ridge_qp_{k}"] for k in olqr.FIELDS})
    sol = olqr.solve(qp)
    assert rel(sol.dx, g["ridge_dx"]) <= 1e-8 and rel(sol.K, g["ridge_K"]) <= 1e-8
    with pytest.raises(olqr.SingularStageError, match="^" + str(g["singR_msg"]) + "$"):
        olqr.solve(olqr.QP(**{k: g[f"singR_qp_{k}"] for k in olqr.FIELDS}))
    N, c = g["singQu_A"].shape[0], g["singQu_C"].shape[1]
    nx, nu = g["singQu_A"].shape[-1], g["singQu_D"].shape[-1]
    du = osls.Duals.zero(N, c, 1, 1e-8)
    du.tau = P.unpack_lower(g["singQu_tau"], N, 1, N)
    costs = osls.assemble_costs(du, g["singQu_C"], g["singQu_D"], g["singQu_CN"],
                                osls.Weights(np.eye(nx), -0.5 * np.eye(nu), np.eye(nx)))
    with pytest.raises(olqr.SingularStageError, match=r"^singular Qu block at \(k=3, j=1\)$"):
        osls.synthesize(g["singQu_A"], g["singQu_B"], g["singQu_E"], costs)
    m = M.DubinsCar(obstacles=((1.0, 0.5, 0.3),))
    x = g["nonfinite_x"]
    with pytest.raises(ArithmeticError, match="^" + str(g["nonfinite_msg"]) + "$"):
        osqp.linearize(m, osqp.Trajectory(x, np.zeros((x.shape[0] - 1, 1)), m.dt))
