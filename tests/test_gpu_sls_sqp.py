"""GPU parity: SLS synthesis / tightening / duals, device linearization and the
robust RTI step vs the golden fixtures (real reference) and the CPU oracle.

Tolerance: 1e-4 relative (reference.relative_error) for fp32 device values
against fp64; ADMM iteration counts exactly.
"""

import numpy as np
import pytest

import oracle
from oracle import sls as osls, sqp as osqp
from conftest import load_golden
import problems as P
from paper_2604_07644_b200 import models as M

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def G():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_07644_b200 import sls, sqp
    return sls, sqp


def rel(a, b):
    return oracle.relative_error(a, b)


def _golden_resp(g, prefix, N, nx, nu):
    return (P.unpack_lower(g[prefix + "phix"], N, 1, N + 1), P.unpack_lower(g[prefix + "phiu"], N, 1, N),
            P.unpack_lower(g[prefix + "gain"], N, 1, N))


def test_sls_selftest_golden(G):
    sls, _ = G
    g = load_golden("sls")
    N, nx, nu = 40, 4, 2
    costs = sls.assemble_costs(None, g["C"], g["D"], g["CN"], sls.SlsWeights.identity(nx, nu))
    resp = sls.synthesize(g["A"], g["B"], g["E"], costs)
    px, pu, gn = _golden_resp(g, "r1_", N, nx, nu)
    for j in range(N):
        assert rel(resp.Phi_x[j], px[j]) <= TOL, j
        assert rel(resp.Phi_u[j], pu[j]) <= TOL, j
        assert rel(resp.gains[j], gn[j]) <= TOL, j
    t = sls.tighten(resp, g["C"], g["D"], g["CN"])
    assert rel(t.h, g["h"]) <= TOL and rel(t.hf, g["hf"]) <= TOL
    du = sls.compute_duals(g["lam_s"], g["lam_t"], resp, g["C"], g["D"], g["CN"], 1e-6)
    assert rel(P.pack_lower(du.tau, N, 1, N, (2,)), g["tau"]) <= TOL
    assert rel(du.tau_term, g["tau_term"]) <= TOL
    w2 = sls.SlsWeights(2 * np.eye(nx), 3 * np.eye(nu), np.eye(nx))
    costs2 = sls.assemble_costs(du, g["C"], g["D"], g["CN"], w2)
    resp2 = sls.synthesize(g["A"], g["B"], g["E"], costs2)
    t2 = sls.tighten(resp2, g["C"], g["D"], g["CN"])
    assert rel(t2.h, g["h2"]) <= TOL and rel(t2.hf, g["hf2"]) <= TOL
    assert sls.sls_cost(resp2, w2) == pytest.approx(float(g["cost2"]), rel=1e-4)


def test_sls_explicit_costs_and_foreign_response(G):
    """synthesize on user-built SlsCosts; tighten on a host-built response (import path)."""
    sls, _ = G
    g = load_golden("sls")
    N, nx, nu = 40, 4, 2
    oc = osls.assemble_costs(None, g["C"], g["D"], g["CN"], osls.Weights.identity(nx, nu))
    costs = sls.SlsCosts(oc.Qx, oc.Qu, oc.Qux, oc.Qx_term)
    resp = sls.synthesize(g["A"], g["B"], g["E"], costs)
    px, pu, gn = _golden_resp(g, "r1_", N, nx, nu)
    assert max(rel(resp.Phi_x[j], px[j]) for j in range(N)) <= TOL
    host = sls.SlsResponse(px, pu, gn, N, nx, nu)
    t = sls.tighten(host, g["C"], g["D"], g["CN"])
    assert rel(t.h, g["h"]) <= TOL


def test_sls_hand_two_stage(G):
    sls, _ = G
    costs = sls.SlsCosts([np.ones((1, 1, 1)), np.zeros((0, 1, 1))], [np.ones((1, 1, 1)), np.zeros((0, 1, 1))],
                         [np.zeros((1, 1, 1)), np.zeros((0, 1, 1))], np.ones((2, 1, 1)))
    ones = np.ones((2, 1, 1))
    r = sls.synthesize(ones, ones, ones, costs)
    assert r.gains[0][0, 0, 0] == pytest.approx(-0.5, abs=1e-6)
    assert r.phi_x(2, 0)[0, 0] == pytest.approx(0.5, abs=1e-6)
    assert r.phi_u(1, 0)[0, 0] == pytest.approx(-0.5, abs=1e-6)


def test_sls_vs_sequential_random(G):
    sls, _ = G
    rng = np.random.default_rng(7)
    N, nx, nu, c = 12, 6, 3, 4
    A = rng.standard_normal((N, nx, nx)) * 0.3 + np.eye(nx)
    A /= np.linalg.norm(A, 2, axis=(1, 2), keepdims=True)
    B = rng.standard_normal((N, nx, nu)) * 0.5
    E = rng.standard_normal((N, nx, nx)) * 0.05
    C = rng.standard_normal((N, c, nx))
    D = rng.standard_normal((N, c, nu))
    CN = rng.standard_normal((2, nx))
    w = osls.Weights.identity(nx, nu)
    oc = osls.assemble_costs(None, C, D, CN, w)
    seq = osls.fastsls_sequential(A, B, E, oc)
    resp = sls.synthesize(A, B, E, sls.assemble_costs(None, C, D, CN, sls.SlsWeights.identity(nx, nu)))
    for j in range(N):
        assert rel(resp.Phi_x[j], seq.Phi_x[j]) <= TOL
        assert rel(resp.Phi_u[j], seq.Phi_u[j]) <= TOL


@pytest.mark.parametrize("model", [
    M.DubinsCar(obstacles=((1.0, 0.5, 0.3),)),
    M.PlanarQuadrotor(obstacles=((1.5, 0.0, 0.35),)),
    M.NLinkPendulum(n_links=3, e_rate=0.05),
    M.Quadrotor12(),
    M.quadruped61(),
])
def test_device_linearize_matches_host_model(G, model):
    _, sqp = G
    rng = np.random.default_rng(1)
    N = 6
    x = rng.standard_normal((N + 1, model.nx)) * 0.2
    u = rng.standard_normal((N, model.nu)) * 0.5
    traj = osqp.Trajectory(x, u, model.dt)
    tight = osls.Tightening(np.abs(rng.standard_normal((N, model.nc))) * 0.1,
                            np.abs(rng.standard_normal(model.nf)) * 0.1)
    xb = x[0] + 0.01
    ref = osqp.linearize(model, traj, tight, xb)
    got = sqp.linearize(model, sqp.Trajectory(x, u, model.dt), tight, xb)
    for fld in ("A", "B", "b", "Q", "R", "S", "q", "r", "QN", "qN", "C", "D", "f", "CN", "fN", "dx0"):
        assert rel(getattr(got, fld), getattr(ref, fld)) <= 1e-5, fld


def _rti_case(tag):
    import test_oracle_golden as T
    return T.rti_case(tag)


def _to_ours(sls, sqp, rs):
    from paper_2604_07644_b200 import admm
    a = rs.sqp.admm
    st = sqp.SqpSettings(max_sqp_iters=rs.sqp.max_sqp_iters, kkt_tol=rs.sqp.kkt_tol,
                         admm=admm.AdmmSettings(rho0=a.rho0, rho_min=a.rho_min, rho_max=a.rho_max, sigma=a.sigma,
                                                tol_primal=a.tol_primal, tol_dual=a.tol_dual, max_iter=a.max_iter))
    w = rs.weights
    return sls.RobustSettings(sqp=st, weights=sls.SlsWeights(w.Qbar, w.Rbar, w.QbarN), eps=rs.eps)


@pytest.mark.parametrize("tag", ["pq", "q61", "h75"])
def test_rti_robust_step_golden(G, tag):
    """The drop-in sls.rti_robust_step vs the reference: ADMM iterations, rho changes and
    the active set exactly (pq terminates on its own residual test at 661 iterations, not
    on max_iter); every output within 1e-4."""
    sls, sqp = G
    import test_oracle_golden as T
    from paper_2604_07644_b200 import admm
    g = load_golden("rti")
    model, rs = _rti_case(tag)
    x, prev, tau = T.rti_inputs(g, tag, model)
    ours = _to_ours(sls, sqp, rs)
    t_ours = None
    if tau is not None:
        t_ours = sls.SlsDuals(tau.tau, tau.tau_term, tau.beta, tau.beta_term, tau.eps)
    N = prev.N
    st = admm.AdmmState.fresh(N * model.nc + model.nf, ours.sqp.admm.rho0)
    r = sls.rti_robust_step(model, x, sqp.Trajectory(prev.x, prev.u, prev.dt), t_ours, ours, warm_admm=st)
    assert r.stats.admm_iterations == int(g[f"{tag}_admm_iters"])
    assert r.stats.converged   # every golden step terminated on its residual test
    assert st.generation == int(g[f"{tag}_rho_changes"])
    # active set: z = min(G + y, f) against the offsets the device ADMM used, i.e. the
    # device linearization tightened by the device h (the golden's f differs in the last bits)
    qp = sqp.linearize(model, sqp.Trajectory(prev.x, prev.u, prev.dt), r.tightening, x)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    assert ((st.z >= f - 1e-12) == g[f"{tag}_active"]).all()
    assert rel(r.tightening.h, g[f"{tag}_h"]) <= TOL
    assert rel(r.tightening.hf, g[f"{tag}_hf"]) <= TOL
    assert rel(r.u0, g[f"{tag}_u0"]) <= TOL
    assert rel(r.plan.x, g[f"{tag}_plan_x"]) <= TOL
    assert rel(r.plan.u, g[f"{tag}_plan_u"]) <= TOL
    assert rel(r.lam_stage, g[f"{tag}_lam_s"]) <= TOL
    assert rel(r.lam_terminal, g[f"{tag}_lam_t"]) <= TOL
    assert rel(P.pack_lower(r.tau.tau, N, 1, N, (model.nc,)), g[f"{tag}_tau_out"]) <= TOL
    assert rel(r.tau.tau_term, g[f"{tag}_tau_term_out"]) <= TOL


def test_batched_engine_matches_single(G):
    """A batch of perturbed instances equals the same instances solved one by one."""
    sls, sqp = G
    import torch
    import test_oracle_golden as T
    from paper_2604_07644_b200.engine import RtiEngine
    g = load_golden("rti")
    model, rs = _rti_case("q61")
    x, prev, tau = T.rti_inputs(g, "q61", model)
    ours = _to_ours(sls, sqp, rs)
    B = 4
    rng = np.random.default_rng(0)
    xs = x[None] + 0.002 * rng.standard_normal((B, model.nx)) * (np.arange(B)[:, None] > 0)
    eng = RtiEngine(model, prev.N, B, ours)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    from paper_2604_07644_b200.sls import ragged_to_cells
    tc = np.stack([ragged_to_cells(tau.tau, prev.N, (model.nc,))] * B)
    tt = np.stack([tau.tau_term] * B)
    eng.step(d(xs), d(np.stack([prev.x] * B)), d(np.stack([prev.u] * B)), tau=d(tc), tau_term=d(tt))
    its = eng.stats.iterations.cpu().numpy()
    u0 = eng.u0.cpu().numpy()
    assert its[0] == int(g["q61_admm_iters"])
    assert rel(u0[0], g["q61_u0"]) <= TOL
    for i in range(1, B):
        r = sls.rti_robust_step(model, xs[i], sqp.Trajectory(prev.x, prev.u, prev.dt),
                                sls.SlsDuals(tau.tau, tau.tau_term, tau.beta, tau.beta_term, tau.eps), ours)
        assert r.stats.admm_iterations == its[i]
        assert np.abs(r.u0 - u0[i]).max() <= 1e-9


def test_solve_nmpc_planar_quadrotor_vs_oracle(G):
    _, sqp = G
    from paper_2604_07644_b200 import admm
    model = M.PlanarQuadrotor(dt=0.05, thrust_max=30.0, goal=(2.6, 0, 0, 0, 0, 0), obstacles=((1.5, 0.0, 0.35),))
    x0 = np.array([0.4, 0.3, 0, 0, 0, 0])
    s = dict(rho0=10.0, tol_primal=1e-4, tol_dual=1e-4, max_iter=1500)
    ref = osqp.solve_nmpc(model, x0, osqp.Settings(max_sqp_iters=30, kkt_tol=1e-3, admm=oracle.admm.Settings(**s)),
                          osqp.initial_guess(model, x0, 20))
    got = sqp.solve_nmpc(model, x0, sqp.SqpSettings(max_sqp_iters=30, kkt_tol=1e-3, admm=admm.AdmmSettings(**s)),
                         sqp.initial_guess(model, x0, 20))
    assert got.stats.converged == ref.stats.converged
    assert got.stats.iterations == ref.stats.iterations
    assert rel(got.trajectory.x, ref.trajectory.x) <= 1e-3


@pytest.mark.parametrize("path", [("staged", "2"), ("staged", "4"), ("staged", "16"), ("legacy", "1"),
                                  ("staged-forced", "1")])
@pytest.mark.parametrize("tag", ["q61", "h75"])
def test_rti_robust_step_every_replay_path(G, tag, path, monkeypatch):
    """Both ADMM replay kernels (k_admm_staged on clusters of 2..16 CTAs, k_replay with one
    CTA per instance) reproduce the reference's robust RTI step: exact ADMM iteration count,
    u0 / plan within 1e-4."""
    sls, sqp = G
    import test_oracle_golden as T
    kind, cs = path
    monkeypatch.setenv("GSLS_REPLAY_CLUSTER", cs)
    monkeypatch.setenv("GSLS_REPLAY_STAGED", "0" if kind == "legacy" else ("1" if kind == "staged-forced" else "x"))
    g = load_golden("rti")
    model, rs = _rti_case(tag)
    x, prev, tau = T.rti_inputs(g, tag, model)
    ours = _to_ours(sls, sqp, rs)
    t_ours = sls.SlsDuals(tau.tau, tau.tau_term, tau.beta, tau.beta_term, tau.eps)
    r = sls.rti_robust_step(model, x, sqp.Trajectory(prev.x, prev.u, prev.dt), t_ours, ours)
    assert r.stats.admm_iterations == int(g[f"{tag}_admm_iters"])
    assert rel(r.u0, g[f"{tag}_u0"]) <= TOL
    assert rel(r.plan.x, g[f"{tag}_plan_x"]) <= TOL


def test_large_batch_one_cta_per_instance_matches_single(G):
    """B = 160 > 148 / 2 runs k_replay with one CTA per instance (the batched-throughput
    path); sampled instances equal the same instances solved alone (cluster path)."""
    sls, sqp = G
    import torch
    import test_oracle_golden as T
    from paper_2604_07644_b200.engine import RtiEngine
    from paper_2604_07644_b200.sls import ragged_to_cells
    g = load_golden("rti")
    model, rs = _rti_case("q61")
    x, prev, tau = T.rti_inputs(g, "q61", model)
    ours = _to_ours(sls, sqp, rs)
    B = 160
    rng = np.random.default_rng(7)
    xs = x[None] + 0.002 * rng.standard_normal((B, model.nx)) * (np.arange(B)[:, None] > 0)
    eng = RtiEngine(model, prev.N, B, ours)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    tc = np.stack([ragged_to_cells(tau.tau, prev.N, (model.nc,))] * B)
    tt = np.stack([tau.tau_term] * B)
    eng.step(d(xs), d(np.stack([prev.x] * B)), d(np.stack([prev.u] * B)), tau=d(tc), tau_term=d(tt))
    its = eng.stats.iterations.cpu().numpy()
    u0 = eng.u0.cpu().numpy()
    assert its[0] == int(g["q61_admm_iters"])
    assert rel(u0[0], g["q61_u0"]) <= TOL
    for i in (1, 77, 159):
        r = sls.rti_robust_step(model, xs[i], sqp.Trajectory(prev.x, prev.u, prev.dt),
                                sls.SlsDuals(tau.tau, tau.tau_term, tau.beta, tau.beta_term, tau.eps), ours)
        assert r.stats.admm_iterations == its[i]
        assert np.abs(r.u0 - u0[i]).max() <= 1e-9
