"""GPU parity of the BENCHED workload: the batched robust RTI step (cfg-D, 61D/12u, and
E-RTI, 75D/19u) against the REAL reference instance by instance.

tests/golden/batch.npz holds the reference's sls.rti_robust_step (sls.py:500-525) on
scenarios 0..63 (q61) and 0..15 (h75) of paper_2604_07644_b200.scenarios — the same
scenario generator bench.py times.  One batched RtiEngine step (the C-ABI path the
bench measures) must give, for every instance: the ADMM iteration count, the number of
rho changes and the active set exactly; u0, plan, h, hf, lambda, tau within 1e-4
relative (reference.relative_error).  The nominal sqp.rti_step (sqp.py:272-302) through
RtiEngine(robust=False) is checked the same way against tests/golden/nominal.npz.
"""

import numpy as np
import pytest

import oracle
import problems as P
from conftest import load_golden

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return oracle.relative_error(a, b)


def _engine_step(tag, count, robust=True):
    import torch
    from paper_2604_07644_b200 import scenarios as S
    from paper_2604_07644_b200.engine import RtiEngine
    from paper_2604_07644_b200.sls import ragged_to_cells
    wl = S.rti_workload(tag)
    m, N = wl.model, wl.N
    settings = S.our_settings()(m)
    eng = RtiEngine(m, N, count, settings if robust else settings.sqp, robust=robust)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")  # noqa: E731
    xs = wl.scenario_states(0, count)
    px = np.broadcast_to(wl.prev_x, (count,) + wl.prev_x.shape)
    pu = np.broadcast_to(wl.prev_u, (count,) + wl.prev_u.shape)
    if robust:
        tc = np.broadcast_to(ragged_to_cells(wl.tau, N, (m.nc,)), (count, N * (N + 1) // 2, m.nc))
        tt = np.broadcast_to(wl.tau_term, (count, N, m.nf))
        eng.step(d(xs), d(px), d(pu), tau=d(tc), tau_term=d(tt))
    else:
        eng.step(d(xs), d(px), d(pu))
    torch.cuda.synchronize()
    return eng, wl, xs


def _host(t):
    return t.detach().cpu().numpy()


def _active(eng):
    f = np.concatenate([_host(eng.qp.f).reshape(eng.B, -1), _host(eng.qp.fN)], axis=1)
    return _host(eng.state.z) >= f - 1e-12


@pytest.mark.parametrize("tag,count", [("q61", 64), ("h75", 16)])
def test_batched_robust_step_matches_reference_per_instance(tag, count):
    g = load_golden("batch")
    eng, wl, xs = _engine_step(tag, count)
    m, N = wl.model, wl.N
    assert np.abs(xs - g[f"{tag}_x"]).max() == 0.0, "scenario generator drifted from the fixture"
    its = _host(eng.stats.iterations)
    rc = _host(eng.stats.rho_changes)
    conv = _host(eng.stats.converged).astype(bool)
    act = _active(eng)
    from paper_2604_07644_b200.sls import cells_to_ragged
    tau = _host(eng.tau)
    bad = []
    for i in range(count):
        ok = (its[i] == g[f"{tag}_iters"][i] and rc[i] == g[f"{tag}_rho_changes"][i]
              and conv[i] == g[f"{tag}_converged"][i] and (act[i] == g[f"{tag}_active"][i]).all())
        if not ok:
            bad.append((i, int(its[i]), int(g[f"{tag}_iters"][i]), int((act[i] != g[f"{tag}_active"][i]).sum())))
    assert not bad, f"instances with a different ADMM path (i, ours, ref, active diffs): {bad}"
    for i in range(count):
        assert rel(_host(eng.u0[i]), g[f"{tag}_u0"][i]) <= TOL, i
        assert rel(_host(eng.h[i]), g[f"{tag}_h"][i]) <= TOL, i
        assert rel(_host(eng.hf[i]), g[f"{tag}_hf"][i]) <= TOL, i
        assert rel(_host(eng.state.lam[i]), g[f"{tag}_lam"][i].astype(float)) <= TOL, i
        assert rel(_host(eng.plan_x[i]), g[f"{tag}_plan_x"][i].astype(float)) <= TOL, i
        assert rel(_host(eng.plan_u[i]), g[f"{tag}_plan_u"][i].astype(float)) <= TOL, i
        t_ours = P.pack_lower(cells_to_ragged(tau[i], N, 1, N), N, 1, N, (m.nc,))
        assert rel(t_ours, g[f"{tag}_tau"][i].astype(float)) <= TOL, i
        assert rel(_host(eng.tau_term[i]), g[f"{tag}_tau_term"][i]) <= TOL, i


@pytest.mark.parametrize("tag,ref_count", [("q61", 64), ("h75", 16)])
def test_large_batch_one_cta_per_instance_matches_reference(tag, ref_count):
    """At 256 instances the ADMM runs one CTA per instance (k_admm_staged with item groups,
    z / lam / y in global memory; the benched configuration) instead of the small-batch
    clusters: its first instances are the fixture's scenarios and must reproduce the
    reference exactly (iterations, rho changes, active set) and within 1e-4."""
    count = 256
    g = load_golden("batch")
    eng, wl, xs = _engine_step(tag, count)
    assert np.abs(xs[:ref_count] - g[f"{tag}_x"]).max() == 0.0
    its, rc = _host(eng.stats.iterations), _host(eng.stats.rho_changes)
    act = _active(eng)
    bad = [i for i in range(ref_count) if not (its[i] == g[f"{tag}_iters"][i] and rc[i] == g[f"{tag}_rho_changes"][i]
                                                and (act[i] == g[f"{tag}_active"][i]).all())]
    assert not bad, bad
    for i in range(ref_count):
        assert rel(_host(eng.u0[i]), g[f"{tag}_u0"][i]) <= TOL, i
        assert rel(_host(eng.state.lam[i]), g[f"{tag}_lam"][i].astype(float)) <= TOL, i


def test_batch_fixture_spreads_iterations():
    """The benched scenarios are not near-identical: the reference's iteration counts vary
    (q61: 21..65 for most instances, a heavy tail up to the max_iter = 500 cap)."""
    g = load_golden("batch")
    its = g["q61_iters"]
    assert its.max() - its.min() >= 100
    assert g["q61_converged"].mean() >= 0.9 and g["h75_converged"].mean() >= 0.9


def test_nominal_rti_engine_matches_reference():
    """RtiEngine(robust=False): the nominal sqp.rti_step per instance (sqp.py:272-302)."""
    g = load_golden("nominal")
    count = g["q61_iters"].shape[0]
    eng, wl, xs = _engine_step("q61", count, robust=False)
    its = _host(eng.stats.iterations)
    act = _active(eng)
    for i in range(count):
        assert its[i] == g["q61_iters"][i], (i, its[i], g["q61_iters"][i])
        assert _host(eng.stats.rho_changes)[i] == g["q61_rho_changes"][i]
        assert (act[i] == g["q61_active"][i]).all(), i
        assert rel(_host(eng.u0[i]), g["q61_u0"][i]) <= TOL
        assert rel(_host(eng.plan_x[i]), g["q61_plan_x"][i]) <= TOL
        assert rel(_host(eng.warm_x[i]), g["q61_warm_x"][i]) <= TOL
        assert rel(_host(eng.state.lam[i]), g["q61_lam"][i]) <= TOL
        assert abs(float(eng.cost[i]) - g["q61_cost"][i]) <= TOL * max(1.0, abs(g["q61_cost"][i]))


def test_nominal_rti_step_dropin_matches_reference():
    """sqp.rti_step through the numpy drop-in API, scenario 3."""
    from paper_2604_07644_b200 import admm, scenarios as S, sqp
    g = load_golden("nominal")
    wl = S.rti_workload("q61")
    m = wl.model
    st = sqp.SqpSettings(admm=admm.AdmmSettings(**S.ADMM), **S.SQP)
    x = wl.scenario_states(3, 1)[0]
    r = sqp.rti_step(m, x, sqp.Trajectory(wl.prev_x, wl.prev_u, m.dt), st)
    assert r.stats.admm_iterations == g["q61_iters"][3]
    assert rel(r.u0, g["q61_u0"][3]) <= TOL
    assert rel(r.plan.x, g["q61_plan_x"][3]) <= TOL
    assert rel(r.warm_start.x, g["q61_warm_x"][3]) <= TOL
    assert abs(r.stats.cost - g["q61_cost"][3]) <= TOL * max(1.0, abs(g["q61_cost"][3]))


def test_benched_batch_with_lagged_rebuilds_matches_reference():
    """The benched size (1024 q61 instances): the bulk ADMM waves run with lagged rebuilds
    (GSLS_ADMM_LAG_MIN, default 2 per SM; csrc/admm.cu admm_solve), the rebuilt instances
    rejoining one wave later.  The fixture's instances still follow the reference's ADMM
    path exactly and match it within 1e-4."""
    count, ref_count = 1024, 64
    g = load_golden("batch")
    eng, wl, xs = _engine_step("q61", count)
    assert np.abs(xs[:ref_count] - g["q61_x"]).max() == 0.0
    its, rc = _host(eng.stats.iterations), _host(eng.stats.rho_changes)
    act = _active(eng)
    bad = [i for i in range(ref_count) if not (its[i] == g["q61_iters"][i] and rc[i] == g["q61_rho_changes"][i]
                                                and (act[i] == g["q61_active"][i]).all())]
    assert not bad, bad
    for i in range(ref_count):
        assert rel(_host(eng.u0[i]), g["q61_u0"][i]) <= TOL, i
        assert rel(_host(eng.h[i]), g["q61_h"][i]) <= TOL, i


def test_lagged_rebuilds_keep_every_instance_path(monkeypatch):
    """Every wave lagged (GSLS_ADMM_LAG_MIN=2) against none (=0) at 256 instances: the same
    ADMM iteration counts, rho changes and builds for every instance, and the same results
    up to the summation order of the cluster sizes the waves pick (1e-6 absolute)."""
    out = {}
    for lag in ("0", "2"):
        monkeypatch.setenv("GSLS_ADMM_LAG_MIN", lag)
        eng, _, _ = _engine_step("q61", 256)
        out[lag] = (_host(eng.stats.iterations), _host(eng.stats.rho_changes), _host(eng.stats.cache_builds),
                    _host(eng.u0), _host(eng.state.lam))
    a, b = out["0"], out["2"]
    for k in range(3):
        assert np.array_equal(a[k], b[k]), k
    assert np.abs(a[3] - b[3]).max() <= 1e-6
    assert np.abs(a[4] - b[4]).max() <= 1e-6 * max(1.0, np.abs(a[4]).max())


def test_pack_engine_record_through_the_c_abi():
    """dist.pack_engine (gsls_rti_pack_results): the per-instance record the ranks of a
    multi-GPU bench all-gather after every step is [u0 | iterations, converged, rho
    changes, cost], in instance order; gather_results at world size 1 copies it."""
    import torch
    from paper_2604_07644_b200 import dist as D
    eng, wl, _ = _engine_step("q61", 8)
    rec = _host(D.pack_engine(eng))
    nu = eng.u0.shape[1]
    assert rec.shape == (8, nu + len(D.RESULT_FIELDS))
    assert np.array_equal(rec[:, :nu], _host(eng.u0))
    assert np.array_equal(rec[:, nu], _host(eng.stats.iterations).astype(float))
    assert np.array_equal(rec[:, nu + 1], _host(eng.stats.converged).astype(float))
    assert np.array_equal(rec[:, nu + 2], _host(eng.stats.rho_changes).astype(float))
    assert np.array_equal(rec[:, nu + 3], _host(eng.cost))
    out = torch.empty(8, rec.shape[1], dtype=torch.float64, device="cuda")
    assert np.array_equal(_host(D.gather_results(D.pack_engine(eng), 1, out=out)), rec)
