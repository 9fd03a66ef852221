"""bench.py's multi-rank path end to end on one GPU: two ranks under
torchrun share device 0 with host-staged gloo gathers (DC_BENCH_DEVICE / DC_BENCH_BACKEND
exist for exactly this; no kernel of one rank waits on the other), so the partition, the
(c_i, zeta_i) all-gather, the drifter gather and the rank-0 forecast statistics all run
through the same code as the NCCL path on a multi-GPU box."""
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


def test_bench_two_ranks_one_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DC_BENCH_DEVICE="0", DC_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--members", "6", "--nx", "100", "--ny", "60",
           "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["members_total"] == 12
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] > 6 * 40  # diagnostics + drifters + forecast stats
