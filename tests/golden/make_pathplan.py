"""Golden paths from the LIVE reference: the Example 4 barrier-map
pipeline (E/cli.py:154-187) and a smooth single-source field, each solved by the reference's
``solve_ifim`` and walked by its ``gradient_descent_path`` (E/pathplan.py:274-330).

Run in the authoring container only (the GPU box has no /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pathplan.py

Writes tests/golden/pathplan.json: per case the inputs (map size, seeds, step, query point),
the phi digest of the reference solve, and the path (points, phi) as exact floats."""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import eikonal as E  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    for n, step in ((64, 0.5), (96, 0.25), (160, 0.5)):
        bmap = E.synthetic_barrier_map(n)
        start, goal = E.synthetic_endpoints(n)
        grid = E.new_grid(n, n, 1.0, 1.0, origin=(0.0, 0.0), speed=E.barrier_speed(bmap))
        E.solve_ifim(grid, E.seed_point(grid, start, 0.0))
        q = grid.cell_center(goal.i, goal.j)
        path = E.gradient_descent_path(grid, q, step)
        out[f"example4_n{n}_step{step}"] = {
            "kind": "example4", "n": n, "step": step, "start": list(start), "goal": list(goal), "query": list(q),
            "phi_sha256": sha(grid.phi), "points": [list(p) for p in path.points], "phi": list(path.phi)}
    for n, step, q in ((48, 0.5, (40.0, 7.5)), (80, 1.0, (3.0, 70.0))):
        grid = E.new_grid(n, n, 1.0, 1.0, origin=(0.0, 0.0), speed=1.0)
        c = E.CellIndex(n // 3, n // 2)
        E.solve_ifim(grid, E.seed_point(grid, c, 0.0))
        path = E.gradient_descent_path(grid, q, step)
        out[f"single_n{n}_step{step}"] = {
            "kind": "single", "n": n, "step": step, "start": list(c), "query": list(q),
            "phi_sha256": sha(grid.phi), "points": [list(p) for p in path.points], "phi": list(path.phi)}
    with open(os.path.join(HERE, "pathplan.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print({k: len(v["points"]) for k, v in out.items()})


if __name__ == "__main__":
    main()
