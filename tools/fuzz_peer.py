"""Long randomised parity run of the multi-GPU peer-slab kernels (k_update_mr / k_remedy_mr), with R
z-slab ranks emulated as CTA groups of one cooperative launch on one GPU: ragged 3D grids,
checkerboards / log-normal / uniform speeds, blocked cells, 1-4 seeds (tests/test_gpu_brick.py
generator), R drawn from 2..8 (at most nz / 2).  Every solve is compared with the oracle bit for bit
(phi, every RunStats integer, active_history).  python tools/fuzz_peer.py [count] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import cpu  # noqa: E402
from paper_2106_15869_b200.slab_peer import solve_emulated  # noqa: E402
from test_gpu_brick import _random_problem  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 19)
dev = torch.device("cuda:0")
bad = 0
for t in range(count):
    shape, h, F, seeds, vals = _random_problem(rng)
    nz = shape[0]
    R = int(rng.integers(2, min(8, nz // 2) + 1))
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    ref = cpu.solve_ifim(shape, h, F, seeds, vals, state=state)
    phi, s, _ = solve_emulated(shape, h, torch.as_tensor(F, device=dev), torch.as_tensor(state, device=dev),
                               list(zip(seeds, vals)), R, device=dev)
    o = ref.stats
    ok = np.array_equal(phi.cpu().numpy().view(np.uint64), ref.phi.reshape(shape).view(np.uint64)) and \
        (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy) == \
        (o["iterations"], o["solver_calls"], o["peak_active"], o["peak_remedy"]) and \
        list(s.active_history) == list(ref.active_history)
    if not ok:
        bad += 1
        print("MISMATCH", t, shape, R, h, seeds, flush=True)
print(f"peer-slab fuzz: {count} problems (2..8 emulated ranks), {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
