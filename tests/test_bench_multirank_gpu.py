"""bench.py's multi-rank path (torchrun, slab partition, peer transport, max
over ranks) end to end on the one-GPU box: two ranks share cuda:0 over gloo
(SG_BENCH_ONE_DEVICE=1) and map each other's mailboxes through CUDA IPC."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_bench_two_ranks_peer_transport():
    env = dict(os.environ, SG_BENCH_ONE_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--size", "40"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["converged"]
    assert line["pcg_iters"] == 11  # configs[0] (40^3): the reference's count (tests/golden/cfg40.npz)
    assert "peer transport" in line["config"]["parallelism"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
