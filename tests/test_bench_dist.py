"""bench.py's N>1 paths end to end on one GPU: torchrun with 2-3 ranks sharing
the device, collectives staged through gloo (TFG_DIST_BACKEND=gloo). Checks
that the whole-job GLCMs after halo exchange + one reduce conserve the global
valid-pair counts (the same gate bench.py applies with NCCL on N GPUs)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("wl,n", [("t3", 2), ("t5", 3), ("t4", 2)])
def test_bench_partitioned_layouts(wl, n):
    env = dict(os.environ, TFG_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--workload", wl, "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == n
    assert line["config"]["check"]["conservation"] is True
    assert line["e2e"]["value"] > 0
