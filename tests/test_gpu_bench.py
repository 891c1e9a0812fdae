"""bench.py's multi-rank code path on a one-GPU box (a code-path check, not a measurement).

Two ranks under torch.distributed.run with SS_BENCH_PG=gloo: both on cuda:0 (independent mode
solves, no kernel waits on the other rank), gloo for the timing reductions and the host-staged
field gather.  The JSON line must carry the contract keys with n_gpus = 2.
"""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_code_path():
    env = dict(os.environ, SS_BENCH_PG="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--workload", "c2", "--steps", "1", "--warmup", "1", "--quick", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["value"] > 0
    for key in ("metric", "unit", "ms_per_step", "config", "roofline", "e2e", "gpu_launches", "clocks", "spmv"):
        assert key in line
    assert line["e2e"]["value"] > 0 and "gloo" in line["e2e"]["gather"]
