"""bench.py's N > 1 branch end to end on a one-GPU box: two ranks under torchrun, both on GPU 0
with a gloo process group (test hook OTT_BENCH_ONE_GPU_TEST; the gather is a host-side
collective, so no rank's kernels wait on another's). Each rank shards the (batch x kv-head)
units, runs the timed decode steps and the end-to-end pipeline, and the gathered head outputs
must equal an all-gather of every rank's last-layer rows."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, OTT_BENCH_ONE_GPU_TEST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", "--config", "c3s", "--steps", "3",
           "--warmup", "3", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["partition"].startswith("128 (batch x kv-head) units / 2 rank(s)")
    assert line["gather"].startswith("NCCL all_gather_into_tensor")
    assert line["e2e"]["gathered_output_verified"] is True
    assert line["parity"]["bit_exact"] is True and line["parity"]["max_err_over_tol"] < 1.0
