"""Generate golden fixtures by running the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports ``scanmpc`` from /root/reference/pkg/src (read-only, never shipped),
runs it on seeded inputs and stores inputs + outputs as small ``.npz`` files
next to this script.  The GPU box never reads /root/reference; it only reads
these fixtures.  Every fixture records the reference call it came from.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from scanmpc import admm, lqr, models, reference, rollout, scan, sls, sqp  # noqa: E402

import problems as P  # noqa: E402
from paper_2604_07644_b200 import models as ours  # noqa: E402

EX = scan.SequentialExecutor()
FIELDS = ("A", "B", "b", "Q", "R", "S", "q", "r", "QN", "qN", "C", "D", "f", "CN", "fN", "dx0")


def ref_qp(qp):
    return lqr.LtvQpData(**{k: np.array(getattr(qp, k), float) for k in FIELDS})


def qp_dict(qp, prefix="qp_"):
    return {prefix + k: np.asarray(getattr(qp, k), float) for k in FIELDS}


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}.npz ({os.path.getsize(path) / 1024:.1f} KiB)")


def traj_dict(t, prefix):
    return {prefix + "x": t.x, prefix + "u": t.u, prefix + "dt": np.float64(t.dt)}


def gen_scan():
    rng = np.random.default_rng(5)
    ints = rng.integers(-1000, 1000, size=300)
    fwd = scan.inclusive_scan(ints.tolist(), lambda a, b: a + b, 0)
    rev = scan.inclusive_scan(ints.tolist(), lambda a, b: a + b, 0, direction="reverse")
    mats = rng.standard_normal((7, 2, 2))
    suffix = scan.inclusive_scan(list(mats), lambda a, b: a @ b, np.eye(2), direction="reverse")
    save("scan", ints=ints, fwd=np.array(fwd), rev=np.array(rev), mats=mats, suffix=np.array(suffix),
         depths=np.array([[L, scan.scan_depth(L)] for L in (1, 2, 3, 8, 17, 26, 51, 1000, 2048)]))


def gen_lqr():
    out = {}
    for tag, (nx, nu, N, seed) in {"r6": (6, 3, 64, 0), "r5": (5, 2, 29, 1), "r12": (12, 4, 100, 2),
                                   "r61": (61, 12, 25, 3)}.items():
        qp = P.random_ltv_qp(np.random.default_rng(seed), nx, nu, N)
        sol = lqr.solve(ref_qp(qp), executor=EX)
        # inputs are regenerated from the seed by the tests; store a checksum of them
        out[f"{tag}_dims"] = np.array([nx, nu, N, seed])
        out[f"{tag}_checksum"] = np.float64(sum(float(np.abs(getattr(qp, k)).sum()) for k in FIELDS))
        for fld in ("dx", "du", "K", "k", "p"):
            out[f"{tag}_{fld}"] = getattr(sol, fld)
        out[f"{tag}_P0"] = sol.P[0]
        out[f"{tag}_layers"] = np.int64(sol.scan_layers)
    # cached replay with perturbed linear terms (test_lqr.py:250-260)
    qp = P.random_ltv_qp(np.random.default_rng(1), 5, 2, 29)
    _, cache = lqr.build_cache(ref_qp(qp), executor=EX, generation=0)
    rng = np.random.default_rng(11)
    q, r, qN = rng.standard_normal(qp.q.shape), rng.standard_normal(qp.r.shape), rng.standard_normal(qp.qN.shape)
    fast = lqr.solve_cached(lqr.LqrLinearTerms(q, r, qN), cache, 0, executor=EX)
    out.update(pert_q=q, pert_r=r, pert_qN=qN, pert_dx=fast.dx, pert_du=fast.du, pert_k=fast.k, pert_p=fast.p)
    # scalar analytic + N=0
    s = lqr.solve(ref_qp(P.scalar_qp()), executor=EX)
    out.update(scalar_du=s.du, scalar_dx=s.dx)
    save("lqr", **out)


def gen_admm():
    out = {}
    st = admm.AdmmSettings(rho0=0.1, sigma=10, tol_primal=1e-4, tol_dual=1e-4, max_iter=4000)
    qp = P.double_integrator()
    res = admm.solve_qp(ref_qp(qp), st, executor=EX)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    out.update({f"di_{k}": v for k, v in qp_dict(qp).items()})
    out.update(di_dx=res.dx, di_du=res.du, di_lam=res.state.lam, di_z=res.state.z,
               di_iters=np.int64(res.stats.iterations), di_rho=np.float64(res.stats.rho),
               di_rho_changes=np.int64(res.stats.rho_changes), di_builds=np.int64(res.stats.cache_builds),
               di_active=(res.state.z >= f - 1e-12), di_converged=np.bool_(res.stats.converged))
    # batch of seeded initial offsets (SURVEY §8d cfg-A batch)
    rng = np.random.default_rng(123)
    x0s = rng.uniform(-5, 5, (8, 4))
    its, dxs, dus, acts = [], [], [], []
    for x0 in x0s:
        r2 = admm.solve_qp(ref_qp(P.double_integrator(dx0=x0)), st, executor=EX)
        its.append(r2.stats.iterations); dxs.append(r2.dx); dus.append(r2.du)
        acts.append(r2.state.z >= f - 1e-12)
    out.update(dib_x0=x0s, dib_iters=np.array(its), dib_dx=np.array(dxs), dib_du=np.array(dus),
               dib_active=np.array(acts))
    # random problems vs dense IP (test_admm.py:118-129)
    rng = np.random.default_rng(0)
    st6 = admm.AdmmSettings(tol_primal=1e-6, tol_dual=1e-6)
    for i in range(3):
        qp = P.random_ltv_qp(rng, 4, 2, 12, nc=3, nf=1)
        res = admm.solve_qp(ref_qp(qp), st6, executor=EX)
        H, g, Ai, bi, Ae, be = P.dense_form(qp)
        _, obj, _ = reference.dense_qp(H, g, Ai, bi, Ae, be)
        out.update({f"rnd{i}_{k}": v for k, v in qp_dict(qp).items()})
        out.update({f"rnd{i}_dx": res.dx, f"rnd{i}_du": res.du, f"rnd{i}_lam": res.state.lam,
                    f"rnd{i}_iters": np.int64(res.stats.iterations), f"rnd{i}_obj": np.float64(obj),
                    f"rnd{i}_rho_changes": np.int64(res.stats.rho_changes)})
    save("admm", **out)


def pack_resp(resp, N, nx, nu, prefix):
    return {prefix + "phix": P.pack_lower(resp.Phi_x, N, 1, N + 1, (nx, nx)),
            prefix + "phiu": P.pack_lower(resp.Phi_u, N, 1, N, (nu, nx)),
            prefix + "gain": P.pack_lower(resp.gains, N, 1, N, (nu, nx))}


def gen_sls():
    out = {}
    # the selftest instance (cli.py:499-527)
    rng = np.random.default_rng(0)
    qp = P.selftest_lqr(rng)
    nx, nu, N = 4, 2, 40
    E = rng.standard_normal((N, nx, nx)) * 0.05
    C = rng.standard_normal((N, 2, nx))
    D = rng.standard_normal((N, 2, nu))
    CN = rng.standard_normal((1, nx))
    w = sls.SlsWeights.identity(nx, nu)
    costs = sls.assemble_costs(None, C, D, CN, w)
    resp = sls.synthesize(qp.A, qp.B, E, costs, executor=EX)
    t = sls.tighten(resp, C, D, CN)
    lam_s = np.abs(rng.standard_normal((N, 2))) * (rng.random((N, 2)) > 0.5)
    lam_t = np.abs(rng.standard_normal(1))
    du = sls.compute_duals(lam_s, lam_t, resp, C, D, CN, 1e-6)
    costs2 = sls.assemble_costs(du, C, D, CN, sls.SlsWeights(2 * np.eye(nx), 3 * np.eye(nu), np.eye(nx)))
    resp2 = sls.synthesize(qp.A, qp.B, E, costs2, executor=EX)
    t2 = sls.tighten(resp2, C, D, CN)
    out.update(A=qp.A, B=qp.B, E=E, C=C, D=D, CN=CN, lam_s=lam_s, lam_t=lam_t, h=t.h, hf=t.hf,
               tau=P.pack_lower(du.tau, N, 1, N, (2,)), tau_term=du.tau_term,
               beta=P.pack_lower(du.beta, N, 1, N, (2,)), beta_term=du.beta_term,
               h2=t2.h, hf2=t2.hf, cost2=np.float64(sls.sls_cost(resp2, sls.SlsWeights(2 * np.eye(nx), 3 * np.eye(nu), np.eye(nx)))))
    out.update(pack_resp(resp, N, nx, nu, "r1_"))
    out.update(pack_resp(resp2, N, nx, nu, "r2_"))
    # hand 2-stage scalar (test_reference.py:86-98)
    save("sls", **out)


def gen_models():
    rng = np.random.default_rng(4)
    out = {}
    cases = {"dubins": (models.DubinsCar(obstacles=((1.0, 0.5, 0.3),)), ours.DubinsCar(obstacles=((1.0, 0.5, 0.3),))),
             "quad": (models.PlanarQuadrotor(obstacles=((1.5, 0.0, 0.35),)), ours.PlanarQuadrotor(obstacles=((1.5, 0.0, 0.35),))),
             "pend2": (models.NLinkPendulum(n_links=2), ours.NLinkPendulum(n_links=2)),
             "pend4": (models.NLinkPendulum(n_links=4, e_rate=0.05), ours.NLinkPendulum(n_links=4, e_rate=0.05))}
    for tag, (ref, _) in cases.items():
        xs = rng.standard_normal((5, ref.nx)) * 0.5
        us = rng.standard_normal((5, ref.nu))
        out[f"{tag}_x"], out[f"{tag}_u"] = xs, us
        out[f"{tag}_step"] = np.array([ref.step(x, u) for x, u in zip(xs, us)])
        out[f"{tag}_A"] = np.array([ref.jacobians(x, u)[0] for x, u in zip(xs, us)])
        out[f"{tag}_B"] = np.array([ref.jacobians(x, u)[1] for x, u in zip(xs, us)])
        out[f"{tag}_g"] = np.array([ref.stage_constraints(x, u) for x, u in zip(xs, us)])
        out[f"{tag}_C"] = np.array([ref.stage_constraint_jacobians(x, u)[0] for x, u in zip(xs, us)])
        out[f"{tag}_D"] = np.array([ref.stage_constraint_jacobians(x, u)[1] for x, u in zip(xs, us)])
        out[f"{tag}_E"] = np.array([ref.disturbance(x) for x in xs])
        out[f"{tag}_gf"] = np.array([ref.terminal_constraints(x) for x in xs]).reshape(5, -1)
    save("models", **out)


def _rti_with_active(model, x, warm, tau, rs):
    """rti_robust_step with an explicit fresh AdmmState: identical to warm_admm=None
    (admm.py:164 builds the same fresh state), but the reference mutates it in place,
    so its final z gives the active set z >= f (f = the tightened offsets)."""
    nc, nf, N = model.nc, model.nf, warm.N
    st = admm.AdmmState.fresh(N * nc + nf, rs.sqp.admm.rho0)
    r = sls.rti_robust_step(model, x, warm, tau, rs, executor=EX, warm_admm=st)
    qp = sqp.linearize(model, warm, r.tightening, x)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    r.stats.rho_changes_ = _rho_changes(st)
    return r, st.z >= f - 1e-12


def _rho_changes(st):
    return st.generation


def _rti_case(model, x0, N, st, rs, steps, tag, out):
    nom = sqp.solve_nmpc(model, x0, st, sqp.initial_guess(model, x0, N, "rollout"), executor=EX)
    warm, tau, u = nom.trajectory.shifted(), None, nom.trajectory.u[0]
    x = np.asarray(x0, float)
    for s in range(steps):
        x = model.step(x, u)
        r, act = _rti_with_active(model, x, warm, tau, rs)
        if s == steps - 1:
            out[f"{tag}_active"] = act
            out[f"{tag}_rho_changes"] = np.int64(r.stats.rho_changes_)
            N_ = warm.N
            out.update(traj_dict(warm, f"{tag}_prev_"))
            out[f"{tag}_xbar0"] = x
            out[f"{tag}_tau_in"] = P.pack_lower(tau.tau, N_, 1, N_, (model.nc,)) if tau else np.zeros(0)
            out[f"{tag}_tau_term_in"] = tau.tau_term if tau else np.zeros(0)
            out[f"{tag}_u0"] = r.u0
            out.update(traj_dict(r.plan, f"{tag}_plan_"))
            out[f"{tag}_h"], out[f"{tag}_hf"] = r.tightening.h, r.tightening.hf
            out[f"{tag}_lam_s"], out[f"{tag}_lam_t"] = r.lam_stage, r.lam_terminal
            out[f"{tag}_tau_out"] = P.pack_lower(r.tau.tau, N_, 1, N_, (model.nc,))
            out[f"{tag}_tau_term_out"] = r.tau.tau_term
            out[f"{tag}_admm_iters"] = np.int64(r.stats.admm_iterations)
            out[f"{tag}_converged"] = np.bool_(r.stats.converged)
            out[f"{tag}_cost"] = np.float64(r.stats.cost)
            print(tag, "admm iters", r.stats.admm_iterations, "converged", r.stats.converged)
        warm, tau, u = r.warm_start, r.tau, r.u0


def gen_rti():
    out = {}
    # planar quadrotor (quadrotor_compare-like), N=20
    quad_ref = models.PlanarQuadrotor(dt=0.05, thrust_max=30.0, goal=(2.6, 0, 0, 0, 0, 0),
                                      obstacles=((1.5, 0.0, 0.35),))
    st = sqp.SqpSettings(max_sqp_iters=50, kkt_tol=5e-4,
                         admm=admm.AdmmSettings(rho0=10.0, tol_primal=2e-5, tol_dual=2e-5, max_iter=1500))
    # max_iter 3000: the golden step terminates on its own residual test (661 iterations)
    st_rti = sqp.SqpSettings(max_sqp_iters=30, kkt_tol=2e-3,
                             admm=admm.AdmmSettings(rho0=10.0, tol_primal=1e-3, tol_dual=1e-3, max_iter=3000))
    rs = sls.RobustSettings(sqp=st_rti, weights=sls.SlsWeights(np.diag([20.0, 20, 1, 4, 4, 0.5]), 0.3 * np.eye(2),
                                                               np.diag([20.0, 20, 1, 4, 4, 0.5])), eps=1e-4)
    x0 = np.array([0.4, 0.3, 0, 0, 0, 0])
    nom = sqp.solve_nmpc(quad_ref, x0, st, sqp.initial_guess(quad_ref, x0, 20), executor=EX)
    print("quad nmpc", nom.stats)
    warm, tau, u, x = nom.trajectory.shifted(), None, nom.trajectory.u[0], x0
    for s in range(3):
        x = quad_ref.step(x, u)
        r, act = _rti_with_active(quad_ref, x, warm, tau, rs)
        if s == 2:
            out["pq_active"] = act
            out["pq_rho_changes"] = np.int64(r.stats.rho_changes_)
            out.update(traj_dict(warm, "pq_prev_"))
            out["pq_xbar0"] = x
            out["pq_tau_in"] = P.pack_lower(tau.tau, 20, 1, 20, (quad_ref.nc,))
            out["pq_tau_term_in"] = tau.tau_term
            out["pq_u0"] = r.u0
            out.update(traj_dict(r.plan, "pq_plan_"))
            out["pq_h"], out["pq_hf"] = r.tightening.h, r.tightening.hf
            out["pq_lam_s"], out["pq_lam_t"] = r.lam_stage, r.lam_terminal
            out["pq_tau_out"] = P.pack_lower(r.tau.tau, 20, 1, 20, (quad_ref.nc,))
            out["pq_tau_term_out"] = r.tau.tau_term
            out["pq_admm_iters"] = np.int64(r.stats.admm_iterations)
            out["pq_converged"] = np.bool_(r.stats.converged)
            print("pq admm iters", r.stats.admm_iterations, r.stats.converged)
        warm, tau, u = r.warm_start, r.tau, r.u0

    # synthetic legged plants (cfg D / E-RTI), N=25, our host model under the reference solver
    for tag, mdl in (("q61", ours.quadruped61()), ("h75", ours.humanoid75())):
        st = sqp.SqpSettings(max_sqp_iters=30, kkt_tol=1e-3,
                             admm=admm.AdmmSettings(rho0=1.0, tol_primal=1e-3, tol_dual=1e-3, max_iter=500))
        rs = sls.RobustSettings(sqp=st, eps=1e-4,
                                weights=sls.SlsWeights(np.eye(mdl.nx), 10 * np.eye(mdl.nu), np.eye(mdl.nx)))
        x0 = np.zeros(mdl.nx)
        x0[0], x0[1] = -0.3, 0.05
        _rti_case(mdl, x0, 25, st, rs, 2, tag, out)
    save("rti", **out)


def gen_rollout():
    """rollout.closed_loop / sample_disturbance / adversarial_rows (rollout.py:41-160) on
    nominal trajectories with a synthesized response (sls.synthesize on the linearization)."""
    out = {}
    cases = {
        "dubins": (models.DubinsCar(obstacles=((1.0, 0.2, 0.3),)), np.array([0.0, 0.0, 0.1]), 20, 0.3),
        "quad": (models.PlanarQuadrotor(obstacles=((1.5, 0.0, 0.35),)), np.array([0.2, 0.1, 0, 0, 0, 0]), 16, 3.0),
        "pend2": (models.NLinkPendulum(n_links=2), np.array([0.3, -0.2, 0.0, 0.0]), 12, 0.5),
        "q61": (ours.quadruped61(), None, 10, 1.0),
    }
    rng = np.random.default_rng(7)
    for tag, (mdl, x0, N, uscale) in cases.items():
        nx, nu = mdl.nx, mdl.nu
        if x0 is None:
            x0 = np.zeros(nx)
            x0[0], x0[1] = -0.3, 0.05
        # nominal: a rollout under small random inputs (dimensionally valid, not optimal)
        u = rng.standard_normal((N, nu)) * 0.1 * uscale
        x = np.zeros((N + 1, nx))
        x[0] = x0
        for k in range(N):
            x[k + 1] = mdl.step(x[k], u[k])
        traj = sqp.Trajectory(x=x, u=u, dt=mdl.dt)
        qp = sqp.linearize(mdl, traj)
        E = np.array([mdl.disturbance(x[k]) for k in range(N)])
        w = sls.SlsWeights.identity(nx, nu)
        costs = sls.assemble_costs(None, qp.C, qp.D, qp.CN, w)
        resp = sls.synthesize(qp.A, qp.B, E, costs, executor=EX)
        tight = sls.tighten(resp, qp.C, qp.D, qp.CN)
        rows = rollout.adversarial_rows(mdl, traj)
        dists = [rollout.sample_disturbance("uniform_ball", nx, N, 11),
                 rollout.sample_disturbance("boundary", nx, N, 12),
                 rollout.sample_disturbance("adversarial", nx, N, 0, rows=rows),
                 rollout.sample_disturbance("uniform_ball", nx, N, 13) * 3.0]   # violates |w| <= 1
        recs = [rollout.closed_loop(mdl, traj, resp, d, tight) for d in dists]
        rec_nt = rollout.closed_loop(mdl, traj, resp, dists[0], None)          # no tube check
        sup = rollout.superposition_check(traj, resp, recs[0].w, recs[0].x)
        out[f"{tag}_x"], out[f"{tag}_u"], out[f"{tag}_N"] = x, u, np.int64(N)
        out[f"{tag}_phiu"] = P.pack_lower(resp.Phi_u, N, 1, N, (nu, nx))
        out[f"{tag}_phix"] = P.pack_lower(resp.Phi_x, N, 1, N + 1, (nx, nx))
        out[f"{tag}_h"], out[f"{tag}_hf"] = tight.h, tight.hf
        out[f"{tag}_rows"] = rows
        out[f"{tag}_dist"] = np.array(dists)
        for f in ("x", "u", "w", "stage_g", "terminal_g", "tube_margin"):
            out[f"{tag}_rec_{f}"] = np.array([getattr(r, f) for r in recs])
        for f in ("safe", "tube_ok", "disturbance_model_violated", "max_w_norm", "min_margin"):
            out[f"{tag}_rec_{f}"] = np.array([getattr(r, f) for r in recs])
        out[f"{tag}_nt_tube_margin"] = rec_nt.tube_margin
        out[f"{tag}_nt_tube_ok"] = np.bool_(rec_nt.tube_ok)
        out[f"{tag}_superposition"] = np.float64(sup)
        print(tag, "safe", [r.safe for r in recs], "tube", [r.tube_ok for r in recs],
              "viol", [r.disturbance_model_violated for r in recs], "sup", sup)
    save("rollout", **out)


def _batch_worker(args):
    """One reference rti_robust_step of scenario `idx` of the cfg-D / E-RTI workload."""
    tag, idx = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2604_07644_b200 import scenarios as S
    wl = S.rti_workload(tag)
    m = wl.model
    st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.ADMM), **S.SQP)
    rs = sls.RobustSettings(sqp=st, eps=S.EPS,
                            weights=sls.SlsWeights(np.eye(m.nx), S.RBAR * np.eye(m.nu), np.eye(m.nx)))
    tau = sls.SlsDuals.zero(wl.N, m.nc, m.nf, S.EPS)
    tau.tau = [np.array(t) for t in wl.tau]
    tau.tau_term = np.array(wl.tau_term)
    x = wl.scenario_states(idx, 1)[0]
    prev = sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    r, act = _rti_with_active(m, x, prev, tau, rs)
    return dict(x=x, iters=r.stats.admm_iterations, converged=r.stats.converged, active=act,
                rho_changes=r.stats.rho_changes_, u0=r.u0, h=r.tightening.h, hf=r.tightening.hf,
                lam=np.concatenate([r.lam_stage.ravel(), r.lam_terminal]), plan_x=r.plan.x, plan_u=r.plan.u,
                tau=P.pack_lower(r.tau.tau, wl.N, 1, wl.N, (m.nc,)), tau_term=r.tau.tau_term)


def gen_batch():
    """The benched cfg-D batch (and E-RTI) through the REAL reference, per instance:
    scenarios 0..63 of q61 and 0..15 of h75 (paper_2604_07644_b200.scenarios)."""
    import multiprocessing as mp
    out = {}
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        for tag, count in (("q61", 64), ("h75", 16)):
            res = pool.map(_batch_worker, [(tag, i) for i in range(count)])
            for k in res[0]:
                arr = np.array([r[k] for r in res])
                if arr.dtype == np.float64 and k in ("plan_x", "plan_u", "tau", "lam"):
                    arr = arr.astype(np.float32)   # 1e-4 checks; keeps the fixture small
                out[f"{tag}_{k}"] = arr
            its = out[f"{tag}_iters"]
            print(tag, "iterations", its.min(), its.max(), its.mean(), "converged", out[f"{tag}_converged"].all())
    save("batch", **out)


class _QpRecorder:
    """Records every admm.solve_qp the reference makes (iterations, convergence, rho changes)."""

    def __init__(self):
        self.calls = []
        self._orig = admm.solve_qp

    def __enter__(self):
        def wrap(*a, **k):
            r = self._orig(*a, **k)
            self.calls.append((r.stats.iterations, int(r.stats.converged), r.stats.rho_changes, r.stats.cache_builds))
            return r
        sqp.admm.solve_qp = wrap
        return self

    def __exit__(self, *exc):
        sqp.admm.solve_qp = self._orig


def gen_cfgb():
    """BASELINE cfg-B: sqp.solve_nmpc of the 12D quadrotor, N=100, 5 obstacles (sqp.py:190-269)."""
    from paper_2604_07644_b200 import scenarios as S
    m = S.cfgb_model()
    N = S.CFGB["N"]
    x0 = S.quad12_start()
    xg, ug = S.hover_guess(m, x0, N)
    st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGB["admm"]), **S.CFGB["sqp"])
    with _QpRecorder() as rec:
        r = sqp.solve_nmpc(m, x0, st, sqp.Trajectory(xg, ug, m.dt), executor=EX)
    print("cfgB", r.stats, "qp calls", len(rec.calls))
    save("cfgb", x=r.trajectory.x, u=r.trajectory.u, lam_s=r.lam_stage, lam_t=r.lam_terminal,
         sqp_iters=np.int64(r.stats.iterations), converged=np.bool_(r.stats.converged),
         residual=np.float64(r.stats.residual), admm_iters=np.int64(r.stats.admm_iterations),
         cost=np.float64(r.stats.cost), qp_calls=np.array(rec.calls), qp_f=r.qp.f, qp_A0=r.qp.A[0])


def gen_cfgc():
    """BASELINE cfg-C: sls.solve_robust on the 12D quadrotor (sls.py:400-469), N=50."""
    from paper_2604_07644_b200 import scenarios as S
    m = S.cfgc_model()
    N = S.CFGC["N"]
    x0 = S.quad12_start()
    xg, ug = S.hover_guess(m, x0, N)
    st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.CFGC["admm"]), **S.CFGC["sqp"])
    rs = sls.RobustSettings(sqp=st, weights=sls.SlsWeights.identity(m.nx, m.nu), eps=S.CFGC["eps"],
                            tol_h=S.CFGC["tol_h"], max_alternations=S.CFGC["max_alternations"])
    with _QpRecorder() as rec:
        r = sls.solve_robust(m, x0, rs, initial=sqp.Trajectory(xg, ug, m.dt), executor=EX)
    print("cfgC", r.stats, "qp calls", len(rec.calls))
    save("cfgc", x=r.trajectory.x, u=r.trajectory.u, h=r.tightening.h, hf=r.tightening.hf,
         lam_s=r.lam_stage, lam_t=r.lam_terminal, alternations=np.int64(r.stats.alternations),
         converged=np.bool_(r.stats.converged), dh=np.float64(r.stats.dh),
         sqp_iters=np.int64(r.stats.sqp_iterations), qp_calls=np.array(rec.calls),
         tau=P.pack_lower(r.duals.tau, N, 1, N, (m.nc,)), tau_term=r.duals.tau_term,
         **pack_resp(r.response, N, m.nx, m.nu, "resp_"))


def gen_cfge():
    """BASELINE cfg-E: admm.solve_qp of the 75D/19u humanoid linearized over N=2047
    (192,493 variables, 81,882 constraints; admm.py:153-203)."""
    from paper_2604_07644_b200 import scenarios as S
    m = S.cfge_model()
    N = S.CFGE["N"]
    x, u = S.cfge_trajectory(m, N)
    qp = sqp.linearize(m, sqp.Trajectory(x, u, m.dt), None, S.cfge_start(m))
    st = admm.AdmmSettings(**S.CFGE["admm"])
    stt = admm.AdmmState.fresh(N * qp.nc + qp.nf, st.rho0)
    import time
    t = time.perf_counter()
    r = admm.solve_qp(qp, st, warm_start=stt, executor=EX)
    print("cfgE", r.stats, "%.1f s" % (time.perf_counter() - t))
    f = np.concatenate([qp.f.ravel(), qp.fN])
    act = r.state.z >= f - 1e-12
    save("cfge", iters=np.int64(r.stats.iterations), converged=np.bool_(r.stats.converged),
         rho_changes=np.int64(r.stats.rho_changes), builds=np.int64(r.stats.cache_builds),
         active=np.packbits(act), n_active=np.int64(act.sum()), dx=r.dx.astype(np.float32),
         du=r.du.astype(np.float32), lam=r.state.lam.astype(np.float32),
         checksum=np.float64(sum(float(np.abs(getattr(qp, k)).sum()) for k in FIELDS)))


def _nominal_worker(args):
    tag, idx = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from paper_2604_07644_b200 import scenarios as S
    wl = S.rti_workload(tag)
    m = wl.model
    st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.ADMM), **S.SQP)
    x = wl.scenario_states(idx, 1)[0]
    prev = sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt)
    ast = admm.AdmmState.fresh(wl.N * m.nc + m.nf, st.admm.rho0)
    r = sqp.rti_step(m, x, prev, st, executor=EX, warm_admm=ast)
    qp = sqp.linearize(m, prev, None, x)
    f = np.concatenate([qp.f.ravel(), qp.fN])
    return dict(iters=r.stats.admm_iterations, converged=r.stats.converged, active=ast.z >= f - 1e-12,
                rho_changes=ast.generation, u0=r.u0, plan_x=r.plan.x, plan_u=r.plan.u, warm_x=r.warm_start.x,
                lam=np.concatenate([r.lam_stage.ravel(), r.lam_terminal]), cost=r.stats.cost)


def gen_nominal():
    """Nominal sqp.rti_step (sqp.py:272-302) on the cfg-D workload, scenarios 0..7."""
    import multiprocessing as mp
    out = {}
    with mp.get_context("spawn").Pool(os.cpu_count()) as pool:
        res = pool.map(_nominal_worker, [("q61", i) for i in range(8)])
    for k in res[0]:
        out[f"q61_{k}"] = np.array([r[k] for r in res])
    print("nominal q61 iterations", out["q61_iters"])
    save("nominal", **out)


def gen_errors():
    """Error paths of the reference (exception class + message) and the ridge branch."""
    out = {}
    # spd_inverse ridge branch (lqr.py:198-216): input 0 is decoupled (B[:, :, 0] = 0, S[:, 0] = 0) and
    # R[3][0, 0] = 1e-12, so the stage-3 Cholesky pivot^2 < 1e-10 and the block is refactored
    # with the 1e-9 ridge instead of raising
    qp = P.random_ltv_qp(np.random.default_rng(21), 4, 2, 12)
    B = qp.B.copy(); B[:, :, 0] = 0.0
    S = qp.S.copy(); S[:, 0, :] = 0.0
    R = qp.R.copy(); R[3] = np.diag([1e-12, 1.0])
    qp = qp.replace(B=B, S=S, R=R)
    sol = lqr.solve(ref_qp(qp), executor=EX)
    out.update({f"ridge_{k}": v for k, v in qp_dict(qp).items()})
    out.update(ridge_dx=sol.dx, ridge_du=sol.du, ridge_K=sol.K, ridge_k=sol.k)
    # a singular R at stage 5 and 8: the reference names stage 5 (lqr.py:204-215)
    qp2 = P.random_ltv_qp(np.random.default_rng(22), 4, 2, 12)
    R2 = qp2.R.copy(); R2[5] = -np.eye(2); R2[8] = -np.eye(2)
    qp2 = qp2.replace(R=R2)
    try:
        lqr.solve(ref_qp(qp2), executor=EX)
        raise SystemExit("expected SingularStageError")
    except lqr.SingularStageError as e:
        out["singR_msg"] = np.array(str(e))
    out.update({f"singR_{k}": v for k, v in qp_dict(qp2).items()})
    # SLS input-cost block singular at (k=3, j=1) only: Rbar = -0.5 I, and tau weights the
    # D rows of every other valid cell (D' tau D >= 2 I there); _locate_singular names the
    # first failing (k, j) in row-major order (sls.py:258-261, :321-326)
    rng = np.random.default_rng(23)
    N, nx, nu, c = 6, 3, 2, 2
    A = np.tile(np.eye(nx), (N, 1, 1)) + 0.05 * rng.standard_normal((N, nx, nx))
    Bm = rng.standard_normal((N, nx, nu))
    E = 0.1 * np.tile(np.eye(nx), (N, 1, 1))
    C = rng.standard_normal((N, c, nx))
    D = np.tile(np.eye(nu), (N, 1, 1))
    CN = rng.standard_normal((1, nx))
    du = sls.SlsDuals.zero(N, c, 1, 1e-8)
    for j in range(N):
        for k in range(j + 1, N):
            du.tau[j][k - j - 1] = 0.0 if (k, j) in ((3, 1), (4, 2)) else 3.0
    costs = sls.assemble_costs(du, C, D, CN, sls.SlsWeights(np.eye(nx), -0.5 * np.eye(nu), np.eye(nx)))
    try:
        sls.synthesize(A, Bm, E, costs, executor=EX)
        raise SystemExit("expected SingularStageError")
    except lqr.SingularStageError as e:
        out["singQu_msg"] = np.array(str(e))
    out.update(singQu_A=A, singQu_B=Bm, singQu_E=E, singQu_C=C, singQu_D=D, singQu_CN=CN,
               singQu_tau=P.pack_lower(du.tau, N, 1, N, (c,)))
    # non-finite dynamics: x[5] = nan -> the reference names stage 5 (sqp.py:125-126)
    m = models.DubinsCar(obstacles=((1.0, 0.5, 0.3),))
    x = np.zeros((9, 3)); x[:, 0] = np.linspace(0, 1, 9); x[5, 2] = np.nan
    try:
        sqp.linearize(m, sqp.Trajectory(x, np.zeros((8, 1)), m.dt))
        raise SystemExit("expected ArithmeticError")
    except ArithmeticError as e:
        out["nonfinite_msg"] = np.array(str(e))
    out["nonfinite_x"] = x
    for k in ("singR_msg", "singQu_msg", "nonfinite_msg"):
        print(k, out[k])
    save("errors", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["scan", "lqr", "admm", "sls", "models", "rti", "rollout", "batch", "cfgb", "cfgc",
                             "cfge", "errors", "nominal"]
    for w in which:
        globals()["gen_" + w]()
