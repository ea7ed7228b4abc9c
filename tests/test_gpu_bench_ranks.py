"""bench.py under torchrun at world size 2 on one GPU (gloo for the collectives,
GSLS_BENCH_BACKEND=gloo): the multi-rank control flow the driver's scaling run uses —
barriers around the timed loops, the max-over-ranks time, the per-step all-gather of the
result records, the ranks other than 0 leaving before rank 0's diagnostic passes — ends
with exit code 0 and exactly one JSON line, from rank 0, with the whole-job value.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_prints_one_line():
    env = dict(os.environ, GSLS_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps",
           "2", "--warmup", "3", "--batch", "32", "--no-latency", "--no-cpu", "--rh-steps", "5"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 2 and d["config"]["batch_per_gpu"] == 32
    assert d["value"] > 0 and abs(d["value"] - 2 * 32 * 2 / (d["ms_per_step"] * 2 / 1e3)) <= 1e-6 * d["value"]
    assert d["parity"] is None and d["cpu_baseline"] is None  # both are N = 1 only
