"""Long randomised parity run (tests/test_gpu_fuzz.py generator): python tools/fuzz_parity.py [count] [seed]."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402
from oracle import cpu  # noqa: E402
from test_gpu_fuzz import _bc, _grid, _problem  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 500
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = 0
for t in range(count):
    shape, spacing, F, seeds, vals = _problem(rng)
    state = np.where(F == 0, 4, 0).astype(np.uint8)
    ref = cpu.solve_ifim(shape, spacing, F, seeds, vals, state=state, threads=1)
    g = _grid(shape, spacing, F, state)
    res = eik.solve_ifim(g, _bc(shape, seeds, vals))
    ok = np.array_equal(np.asarray(res.phi).view(np.uint64), ref.phi.view(np.uint64)) and \
        res.stats.solver_calls == ref.stats["solver_calls"] and res.stats.active_history == ref.active_history
    fr = cpu.solve_fim(shape, spacing, F, seeds, vals, state=state)
    fg = eik.solve_fim(_grid(shape, spacing, F, state), _bc(shape, seeds, vals))
    ok = ok and np.array_equal(np.asarray(fg.phi).view(np.uint64), fr.phi.view(np.uint64)) and \
        fg.stats.solver_calls == fr.stats["solver_calls"]
    if not ok:
        bad += 1
        print("MISMATCH", t, shape, spacing, seeds, vals, flush=True)
print(f"{count} problems, {bad} mismatches", flush=True)
