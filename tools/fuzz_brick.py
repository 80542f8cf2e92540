"""Long randomised parity run of the TMA brick remedy engine (tests/test_gpu_brick.py generator:
ragged 3D grids, checkerboards / log-normal / uniform speeds, blocked cells, 1-4 seeds):
python tools/fuzz_brick.py [count] [seed].  Every solve runs with EIK_REMEDY=brick and is compared
with the oracle bit for bit (phi, every RunStats integer, active_history)."""
import os
import sys

os.environ["EIK_REMEDY"] = "brick"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402
from oracle import cpu  # noqa: E402
from paper_2106_15869_b200 import _native  # noqa: E402
from test_gpu_brick import _random_problem  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 500
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 11)
bad = ran = 0
for t in range(count):
    shape, h, F, seeds, vals = _random_problem(rng)
    nz, ny, nx = shape
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    ref = cpu.solve_ifim(shape, h, F, seeds, vals, state=state)
    g = eik.Grid3D(nx, ny, nz, h, (0.0, 0.0, 0.0), np.full(shape, np.inf), F.copy(), state.copy())
    bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v)
                                     for c, v in zip(seeds, vals)))
    res = eik.solve_ifim(g, bc)
    if res.stats.peak_remedy:
        ran += _native.last_remedy_engine() == "brick"
    s, o = res.stats, ref.stats
    ok = np.array_equal(res.phi.view(np.uint64), ref.phi.view(np.uint64)) and \
        (s.iterations, s.solver_calls, s.peak_active, s.peak_remedy, s.phi_writes) == \
        (o["iterations"], o["solver_calls"], o["peak_active"], o["peak_remedy"], o["phi_writes"]) and \
        list(s.active_history) == list(ref.active_history)
    if not ok:
        bad += 1
        print("MISMATCH", t, shape, h, seeds, flush=True)
print(f"brick fuzz: {count} problems, {ran} through the brick engine, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
