"""One disturbance-column shard of the cfg-E SLS synthesis on one GPU:
75D/19u humanoid, N = 2047, the shard [j0, j1) of a `world`-way cell-balanced split
(dist.column_shards).  The full synthesis (~2.1M cells) needs ~354 GB; one rank of an
8-way split holds 1/8 of it.  Reports the shard's cells, device memory and the time of
assemble_costs -> synthesize -> tighten (device-side costs, unweighted: tau = None).

    python tools/probe/sls_shard_at_scale.py [world] [rank]
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2604_07644_b200 import _native as nat, dist, scenarios as S  # noqa: E402
from paper_2604_07644_b200.device import Context, stream_ptr, to_dev  # noqa: E402
from paper_2604_07644_b200.engine import DeviceModel, alloc_qp, linearize_into  # noqa: E402

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = S.cfge_model()
N = S.CFGE["N"]
n, mu, c, nf = m.nx, m.nu, m.nc, m.nf
j0, j1 = dist.column_shards(N, world)[rank]
cells = sum(N - j for j in range(j0, j1))
x, u = S.cfge_trajectory(m, N)
free0, total = torch.cuda.mem_get_info()
ctx = Context(n, mu, c, nf, N, 1)
lib = ctx.lib
nat.check(lib.gsls_sls_set_columns(ctx.handle, j0, j1), "columns")
dm = DeviceModel(m, N)
qp = alloc_qp(1, n, mu, c, nf, N)
E = torch.zeros(1, N, n, n, dtype=torch.float32, device="cuda")
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")  # noqa: E731
linearize_into(ctx, dm, qp, d(x[None]), d(u[None]), xbar0=d(S.cfge_start(m)[None]), E=E)
eye = lambda k: to_dev(np.eye(k), torch.float32).contiguous()  # noqa: E731
Qb, Rb, QbN = eye(n), eye(mu), eye(n)
h = torch.zeros(1, N, c, dtype=torch.float64, device="cuda")
hf = torch.zeros(1, nf, dtype=torch.float64, device="cuda")
qs = qp.cstruct()
S_ = stream_ptr()
torch.cuda.synchronize()
t = {}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
t0 = time.perf_counter()
ev[0].record()
nat.check(lib.gsls_sls_assemble(ctx.handle, ctypes.byref(qs), None, None, Qb.data_ptr(), Rb.data_ptr(), QbN.data_ptr(),
                                0, S_), "assemble")
ev[1].record()
nat.check(lib.gsls_sls_synthesize(ctx.handle, ctypes.byref(qs), E.data_ptr(), S_), "synthesize")
ev[2].record()
nat.check(lib.gsls_sls_tighten(ctx.handle, ctypes.byref(qs), h.data_ptr(), hf.data_ptr(), S_), "tighten")
ev[3].record()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
free1, _ = torch.cuda.mem_get_info()
hh = h.cpu().numpy()
out = {"config": "cfg-E SLS shard: 75D/19u humanoid, N=2047, nc=40, nf=2", "world": world, "rank": rank,
       "columns": [j0, j1], "cells": cells, "cells_total": N * (N + 1) // 2,
       "ctx_bytes_GB": ctx.nbytes() / 1e9, "device_used_GB": (free0 - free1) / 1e9, "device_total_GB": total / 1e9,
       "assemble_s": ev[0].elapsed_time(ev[1]) / 1e3, "synthesize_s": ev[1].elapsed_time(ev[2]) / 1e3,
       "tighten_s": ev[2].elapsed_time(ev[3]) / 1e3, "wall_s": wall,
       "h_partial_finite": bool(np.isfinite(hh).all()), "h_partial_min": float(hh.min()),
       "h_partial_max": float(hh.max())}
print(json.dumps(out), flush=True)
