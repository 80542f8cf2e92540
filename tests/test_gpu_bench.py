"""bench.py under torchrun through the fused peer-memory slab path: one rank
per GPU present, `--force-peer` selects `make_peer_step` even at world size 1, and any failure of
the peer path is fatal (no silent switch to the host-driven protocol)."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(*extra, port=29541):
    n = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "2", "--warmup", "3", "--size", "96", "--cpu-size", "16", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    return n, line


def test_bench_peer_step_under_torchrun():
    n, line = _torchrun("--force-peer")
    assert line["n_gpus"] == n and line["value"] > 0
    assert "peer-memory fused kernels" in line["config"]["parallelism"], line["config"]
    assert line["gpu_launches"] > 0


def test_bench_host_slabs_under_torchrun():
    n, line = _torchrun("--force-peer", "--host-slabs", port=29542)
    assert line["n_gpus"] == n and line["value"] > 0
    assert "NCCL" in line["config"]["parallelism"] or "host" in line["config"]["parallelism"], line["config"]
