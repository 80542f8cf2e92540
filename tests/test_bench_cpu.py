"""bench.py contract pieces that run without a GPU: the reference arm's JSON line and the
workload definitions (cfg5 modes/seeds are deterministic)."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-size", "20"], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["config"]["size"] == 512


def test_reference_arm_nonzero_rank_is_silent():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-size", "16"], capture_output=True, text=True, timeout=300,
                         env={**os.environ, "WORLD_SIZE": "2", "RANK": "1"})
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_workloads_are_deterministic():
    import torch

    import bench

    K1, ph1, s1 = bench.cfg5_modes(1024)
    K2, ph2, s2 = bench.cfg5_modes(1024)
    assert np.array_equal(K1, K2) and np.array_equal(ph1, ph2) and s1 == s2
    assert len(K1) == 32 and len(set(map(tuple, K1.tolist()))) == 32 and len(s1) == 16 == len(set(s1))
    assert all(0 < (k * k).sum() <= 16 for k in K1)
    w = bench.make_workload(torch, torch.device("cpu"), "cfg5", 24)
    assert w.F.shape == (24, 24, 24) and float(w.F.min()) > 0 and w.h == 1 / 23
    g = np.log(w.F.numpy()) / 0.5  # unit-variance field (sample variance over the grid, loose check)
    assert 0.3 < g.var() < 3.0
    w4 = bench.make_workload(torch, torch.device("cpu"), "cfg4", 64)
    assert set(np.unique(w4.F.numpy())) == {0.01, 1.0} and w4.seeds == [(32, 32, 32)]
    assert bench.workload_desc("cfg4", 512) == w4.desc.replace("64^3", "512^3").replace("(4^3", "(32^3")
