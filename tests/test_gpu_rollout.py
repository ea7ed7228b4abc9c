"""GPU parity: closed-loop rollouts (rollout.py:47-93) on the device vs the golden
fixtures (real reference) and the CPU oracle.

Tolerance: 1e-4 relative (reference.relative_error) on states, inputs,
reconstructed disturbances, constraint values and tube slack (the device
reads Phi^u in float32); safe / tube_ok / disturbance_model_violated exactly.
"""

import numpy as np
import pytest

import oracle
from oracle import rollout as orl
from conftest import load_golden
import problems as P

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def R():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_07644_b200 import rollout, sls, sqp
    return rollout, sls, sqp


def rel(a, b):
    return oracle.relative_error(a, b)


def _case(g, tag, sls, sqp):
    mdl = P.rollout_model(tag)
    x, u, N = g[f"{tag}_x"], g[f"{tag}_u"], int(g[f"{tag}_N"])
    nx, nu = mdl.nx, mdl.nu
    phiu = P.unpack_lower(g[f"{tag}_phiu"], N, 1, N)
    phix = P.unpack_lower(g[f"{tag}_phix"], N, 1, N + 1)
    resp = sls.SlsResponse(Phi_x=phix, Phi_u=phiu, gains=[p * 0 for p in phiu], N=N, nx=nx, nu=nu)
    tight = sls.Tightening(h=g[f"{tag}_h"], hf=g[f"{tag}_hf"])
    traj = sqp.Trajectory(x=x, u=u, dt=mdl.dt)
    return mdl, traj, resp, tight


def _check_record(r, g, tag, i):
    for f in ("x", "u", "w", "stage_g", "terminal_g"):
        assert rel(getattr(r, f), g[f"{tag}_rec_{f}"][i]) <= TOL, (tag, i, f)
    tm, gtm = r.tube_margin, g[f"{tag}_rec_tube_margin"][i]
    assert np.array_equal(np.isinf(tm), np.isinf(gtm))
    assert rel(np.where(np.isinf(tm), 0, tm), np.where(np.isinf(gtm), 0, gtm)) <= TOL
    assert r.safe == bool(g[f"{tag}_rec_safe"][i]), (tag, i)
    assert r.tube_ok == bool(g[f"{tag}_rec_tube_ok"][i]), (tag, i)
    assert r.disturbance_model_violated == bool(g[f"{tag}_rec_disturbance_model_violated"][i]), (tag, i)
    assert abs(r.max_w_norm - g[f"{tag}_rec_max_w_norm"][i]) <= TOL * max(1.0, r.max_w_norm)
    assert abs(r.min_margin - g[f"{tag}_rec_min_margin"][i]) <= TOL * max(1.0, abs(r.min_margin))


@pytest.mark.parametrize("tag", P.ROLLOUT_TAGS)
def test_rollout_golden(R, tag):
    rollout, sls, sqp = R
    g = load_golden("rollout")
    mdl, traj, resp, tight = _case(g, tag, sls, sqp)
    for i, d in enumerate(g[f"{tag}_dist"]):
        _check_record(rollout.closed_loop(mdl, traj, resp, d, tight), g, tag, i)
    r = rollout.closed_loop(mdl, traj, resp, g[f"{tag}_dist"][0], None)
    assert np.isinf(r.tube_margin).all() and r.tube_ok == bool(g[f"{tag}_nt_tube_ok"])
    sup = rollout.superposition_check(traj, resp, r.w, r.x)
    assert abs(sup - float(g[f"{tag}_superposition"])) <= 1e-6 + TOL * sup
    assert np.array_equal(rollout.adversarial_rows(mdl, traj), g[f"{tag}_rows"]) or \
        rel(rollout.adversarial_rows(mdl, traj), g[f"{tag}_rows"]) <= 1e-9


@pytest.mark.parametrize("tag", ["q61", "dubins"])
def test_rollout_batched_vs_oracle(R, tag):
    """B instances x S rollouts in one launch; every (instance, rollout) against the oracle."""
    import torch
    rollout, sls, sqp = R
    g = load_golden("rollout")
    mdl, traj, resp, tight = _case(g, tag, sls, sqp)
    N, nx, nu, nc = traj.N, mdl.nx, mdl.nu, mdl.nc
    B, S = 3, 8
    rng = np.random.default_rng(5)
    xs = np.stack([traj.x + 0.01 * b * rng.standard_normal(traj.x.shape) for b in range(B)])
    us = np.stack([traj.u + 0.01 * b * rng.standard_normal(traj.u.shape) for b in range(B)])
    hs = np.stack([tight.h * (1.0 + 0.1 * b) for b in range(B)])
    cells = np.stack([sls.ragged_to_cells(resp.Phi_u, N, (nu, nx)) * (1.0 - 0.2 * b) for b in range(B)])
    d = np.stack([[rollout.sample_disturbance("uniform_ball" if s % 2 else "boundary", nx, N, 100 * b + s)
                   * (1.2 if s == 5 else 1.0) for s in range(S)] for b in range(B)])
    dev = lambda a, t=torch.float64: torch.as_tensor(np.ascontiguousarray(a), dtype=t, device="cuda")  # noqa: E731
    out = rollout.closed_loop_batched(mdl, dev(xs), dev(us), dev(cells, torch.float32), dev(d), dev(hs))
    host = {k: v.cpu().numpy() for k, v in out.items()}
    cells32 = cells.astype(np.float32).astype(np.float64)
    for b in range(B):
        for s in range(S):
            ref = orl.closed_loop(mdl, xs[b], us[b],
                                  lambda k, j, b=b: cells32[b][sls.cell_index(N, k, j)], d[b, s], hs[b])
            for f in ("x", "u", "w", "stage_g", "terminal_g"):
                assert rel(host[f][b, s], getattr(ref, f)) <= TOL, (b, s, f)
            assert rel(host["tube_margin"][b, s], ref.tube_margin) <= TOL
            assert bool(host["flags"][b, s, 0]) == ref.safe
            assert bool(host["flags"][b, s, 1]) == ref.tube_ok
            assert bool(host["flags"][b, s, 2]) == ref.disturbance_model_violated
            assert abs(host["max_w_norm"][b, s] - ref.max_w_norm) <= TOL * max(1.0, ref.max_w_norm)
    # open loop (no response) and no tube check
    out = rollout.closed_loop_batched(mdl, dev(xs), dev(us), None, dev(d), None)
    ref = orl.closed_loop(mdl, xs[1], us[1], None, d[1, 3], None)
    assert rel(out["x"][1, 3].cpu().numpy(), ref.x) <= TOL
    assert np.isinf(out["tube_margin"].cpu().numpy()).all()
    assert bool(out["flags"][1, 3, 1].item()) is True


def test_rollout_errors(R):
    rollout, sls, sqp = R
    g = load_golden("rollout")
    mdl, traj, resp, tight = _case(g, "dubins", sls, sqp)
    with pytest.raises(ValueError, match="disturbances must be"):
        rollout.closed_loop(mdl, traj, resp, np.zeros((traj.N + 1, mdl.nx)), tight)
    with pytest.raises(ValueError, match="unknown disturbance kind"):
        rollout.sample_disturbance("cauchy", 3, 4, 0)
