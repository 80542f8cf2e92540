"""Golden fixtures for hand-built RemedySets (E/ifim.py:64-72, :164-218), from the LIVE reference.

The reference's remedy step relaxes ``remedy.cells`` and uses ``remedy.member`` only to decide
which neighbours of a decreased cell get enqueued, so a member outside the work list is never
relaxed and never enqueued, and ``RemedySet(member=m)`` (cells defaults to []) is a no-op.
Writes tests/golden/remedy_sets.npz:

    python tests/golden/make_remedy_sets.py     (authoring container only: needs /root/reference)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from eikonal.grid import CellIndex, new_grid, seed_point  # noqa: E402
from eikonal.ifim import RemedySet, build_remedy_set, ifim_remedy_step, ifim_update_step  # noqa: E402


def main():
    out = {}
    # slow pocket (T/test_ifim.py:43-58): the update step leaves stale values, the build flags them
    sp = np.ones((24, 24))
    sp[8:16, 8:16] = 0.05
    g = new_grid(24, 24, 1.0, 1.0, speed=sp)
    ifim_update_step(g, seed_point(g, CellIndex(0, 0), 0.0))
    remedy, _ = build_remedy_set(g)
    cells = list(remedy.cells)
    out["speed"], out["state"], out["phi_in"] = sp, g.state.copy(), g.phi.copy()
    out["member"] = remedy.member.copy()
    # (a) member-only set: no-op
    g1 = new_grid(24, 24, 1.0, 1.0, speed=sp)
    g1.phi[...] = out["phi_in"]
    g1.state[...] = out["state"]
    st = ifim_remedy_step(g1, RemedySet(member=remedy.member.copy()))
    out["a_stats"] = np.array([st.iterations, st.solver_calls, st.peak_remedy])
    out["a_phi"] = g1.phi.copy()
    # (b) every member marked, every other cell of the work list dropped: members outside the
    # work list block the enqueue of their cells
    work = cells[::2]
    g2 = new_grid(24, 24, 1.0, 1.0, speed=sp)
    g2.phi[...] = out["phi_in"]
    g2.state[...] = out["state"]
    rs = RemedySet(member=remedy.member.copy(), cells=list(work))
    st = ifim_remedy_step(g2, rs)
    out["b_cells"] = np.array(work, dtype=np.int64)
    out["b_stats"] = np.array([st.iterations, st.solver_calls, st.peak_remedy])
    out["b_phi"] = g2.phi.copy()
    out["b_member_after"] = rs.member.copy()
    # (c) plain work list == members (the build's own set)
    g3 = new_grid(24, 24, 1.0, 1.0, speed=sp)
    g3.phi[...] = out["phi_in"]
    g3.state[...] = out["state"]
    st = ifim_remedy_step(g3, RemedySet(member=remedy.member.copy(), cells=list(cells)))
    out["c_stats"] = np.array([st.iterations, st.solver_calls, st.peak_remedy])
    out["c_phi"] = g3.phi.copy()
    np.savez_compressed(os.path.join(HERE, "remedy_sets.npz"), **out)
    print({k: v.tolist() for k, v in out.items() if k.endswith("_stats")})


if __name__ == "__main__":
    main()
