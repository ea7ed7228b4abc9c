"""GPU: SLS with the disturbance columns sharded (gsls_sls_set_columns).

Each shard synthesizes only its columns' cells; its Phi cells must equal the
unsharded synthesis bitwise (columns are independent, sls.py:227-318, and the
merged plan runs the same per-column ops), and the shards' partial tightenings
must sum to the unsharded h, hf (float64 sums in a different order: 1e-9) and
to the real reference's (1e-4).
"""

import numpy as np
import pytest

import oracle
from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    assert torch.cuda.is_available()
    from paper_2604_07644_b200 import dist, sls
    return sls, dist


@pytest.mark.parametrize("world", [2, 3, 5])
def test_sharded_sls_equals_unsharded(S, world):
    sls, dist = S
    g = load_golden("sls")
    A, B, E, C, Dm, CN = (g[k] for k in ("A", "B", "E", "C", "D", "CN"))
    N, nx, nu = A.shape[0], A.shape[1], B.shape[2]
    costs = sls.assemble_costs(None, C, Dm, CN, sls.SlsWeights.identity(nx, nu))
    full = sls.synthesize(A, B, E, costs)
    tf = sls.tighten(full, C, Dm, CN)
    phix_full, phiu_full = (t.cpu().numpy() for t in full._cells[:2])
    h = np.zeros_like(tf.h)
    hf = np.zeros_like(tf.hf)
    for rank, (j0, j1) in enumerate(dist.column_shards(N, world)):
        hp, hfp, phix, phiu = sls.synthesize_tighten_columns(A, B, E, costs, C, Dm, CN, (j0, j1))
        c0 = sls.cell_index(N, j0 + 1, j0)
        assert np.array_equal(phix.cpu().numpy(), phix_full[c0:c0 + phix.shape[0]]), (world, rank)
        assert np.array_equal(phiu.cpu().numpy(), phiu_full[c0:c0 + phiu.shape[0]]), (world, rank)
        h += hp.cpu().numpy()
        hf += hfp.cpu().numpy()
    assert oracle.relative_error(h, tf.h) <= 1e-9
    assert oracle.relative_error(hf, tf.hf) <= 1e-9
    assert oracle.relative_error(h, g["h"]) <= 1e-4
    assert oracle.relative_error(hf, g["hf"]) <= 1e-4


def test_sharded_entry_point_single_rank_and_errors(S):
    sls, dist = S
    g = load_golden("sls")
    A, B, E, C, Dm, CN = (g[k] for k in ("A", "B", "E", "C", "D", "CN"))
    nx, nu = A.shape[1], B.shape[2]
    costs = sls.assemble_costs(None, C, Dm, CN, sls.SlsWeights.identity(nx, nu))
    t, cols, phix, _ = dist.sls_tighten_sharded(A, B, E, costs, C, Dm, CN, rank=0, world=1)
    assert cols == (0, A.shape[0])
    assert oracle.relative_error(t.h, g["h"]) <= 1e-4 and oracle.relative_error(t.hf, g["hf"]) <= 1e-4
    from paper_2604_07644_b200.device import Context
    ctx = Context(nx, nu, C.shape[1], CN.shape[0], A.shape[0], 1)
    assert ctx.lib.gsls_sls_set_columns(ctx.handle, 3, 2) != 0
    assert ctx.lib.gsls_sls_set_columns(ctx.handle, 0, A.shape[0] + 1) != 0
    assert ctx.lib.gsls_sls_set_columns(ctx.handle, 1, 4) == 0
