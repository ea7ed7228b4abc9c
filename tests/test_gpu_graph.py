"""One MPC step as a single CUDA graph (RtiEngine.capture, csrc/admm.cu admm_solve_captured):
the captured step — with the ADMM's rebuild loop as a conditional WHILE node — must give
bitwise the same results as the eager step it records, at batch 1 (cluster replay), at a
small batch, and keep doing so over a receding-horizon sequence of replays.  At a batch
large enough for one CTA per instance (the eager driver then pauses instances in
sigma-aligned waves and the captured loop does not) the iterations, rho changes and builds
are still identical and the values agree to 1e-6."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(tag, B):
    import torch
    from paper_2604_07644_b200 import scenarios as S
    from paper_2604_07644_b200.sls import ragged_to_cells
    wl = S.rti_workload(tag)
    m = wl.model
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")  # noqa: E731
    rep = lambda a: np.broadcast_to(a, (B,) + np.shape(a))  # noqa: E731
    return (wl, d(wl.scenario_states(0, B)), d(rep(wl.prev_x)), d(rep(wl.prev_u)),
            d(rep(ragged_to_cells(wl.tau, wl.N, (m.nc,)))), d(rep(wl.tau_term)))


def _snap(eng):
    return {k: getattr(eng, k).detach().cpu().numpy().copy() for k in ("u0", "plan_x", "plan_u", "h", "tau", "cost")} | {
        "lam": eng.state.lam.cpu().numpy().copy(), "its": eng.stats.iterations.cpu().numpy().copy(),
        "rho_changes": eng.stats.rho_changes.cpu().numpy().copy(),
        "builds": eng.stats.cache_builds.cpu().numpy().copy()}


def _settings(m, rho0):
    import dataclasses
    from paper_2604_07644_b200 import scenarios as S
    rs = S.our_settings()(m)
    if rho0 is not None:  # a small rho0 makes every solve commit rho changes: the WHILE loop iterates
        rs.sqp.admm = dataclasses.replace(rs.sqp.admm, rho0=rho0)
    return rs


@pytest.mark.parametrize("tag,B,rho0", [("q61", 1, None), ("q61", 1, 1e-3), ("q61", 4, 1e-3), ("h75", 1, 1e-3),
                                        ("q61", 200, None)])  # 200: one CTA per instance (4 item groups)
def test_captured_step_equals_eager(tag, B, rho0):
    import torch
    from paper_2604_07644_b200.engine import RtiEngine
    wl, xb, px, pu, tc, tt = _inputs(tag, B)
    m = wl.model
    eager = RtiEngine(m, wl.N, B, _settings(m, rho0))
    ref = []
    eager.step(xb, px, pu, tau=tc, tau_term=tt)
    for _ in range(4):
        eager.step(xb, px, pu)
        torch.cuda.synchronize()
        ref.append(_snap(eager))
    g = RtiEngine(m, wl.N, B, _settings(m, rho0))
    g.step(xb, px, pu, tau=tc, tau_term=tt)
    step = g.capture(xb, px, pu)  # its warm-up is the second eager step
    exact_keys = ("its", "rho_changes", "builds")
    for k in range(1, 4):
        step()
        step.check()
        got = _snap(g)
        for key, v in ref[k].items():
            if B <= 148 or key in exact_keys:
                assert np.array_equal(got[key], v), (k, key)
            else:
                # Above one wave of SMs the eager driver pauses instances at sigma multiples and
                # finishes the long ones on clusters, whose matvecs split k differently from the
                # captured loop's one-CTA launches: the same iterations and decisions, values
                # equal up to the summation order.
                assert np.abs(got[key] - v).max() <= 1e-6 * max(1.0, np.abs(v).max()), (k, key)
    if rho0 is not None:
        assert (ref[-1]["rho_changes"] > 0).all(), "the ADMM rebuild loop was not exercised"


def test_captured_receding_horizon_moves_inputs():
    """New inputs copied into the graph's static buffers each step drive the replay."""
    import torch
    from paper_2604_07644_b200 import scenarios as S
    from paper_2604_07644_b200.engine import RtiEngine
    wl, xb, px, pu, tc, tt = _inputs("q61", 1)
    m = wl.model
    g = RtiEngine(m, wl.N, 1, S.our_settings()(m))
    g.step(xb, px, pu, tau=tc, tau_term=tt)
    step = g.capture(xb, px, pu)
    e = RtiEngine(m, wl.N, 1, S.our_settings()(m))
    e.step(xb, px, pu, tau=tc, tau_term=tt)
    e.step(xb, px, pu)
    x = xb.clone()
    for k in range(5):
        x = x + 1e-3 * (k + 1)
        step(x, g.warm_x.clone(), g.warm_u.clone())
        step.check()
        e.step(x, e.warm_x.clone(), e.warm_u.clone())
        torch.cuda.synchronize()
        assert torch.equal(g.u0, e.u0) and torch.equal(g.plan_x, e.plan_x), k
