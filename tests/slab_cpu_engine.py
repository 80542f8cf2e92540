"""CPU per-rank engine for the slab protocol (paper_2106_15869_b200/slab.py).

Test infrastructure: a direct restatement of E/ifim.py restricted to one z-slab
with ghost planes, using the oracle's bit-exact 3D local solver.  Slow (Python
reconciliation loops), meant for small grids.
"""
import numpy as np
import torch

from oracle import cpu

INF = np.inf
SOURCE, BLOCKED = 2, 4
FAR, ACTIVE, CONVERGED = 0, 1, 2


class CpuSlabEngine:
    def __init__(self, shape, h, speed, state, z0, z1, tol=1e-12):
        nz, ny, nx = shape
        self.nx, self.ny, self.nz = nx, ny, nz
        self.z0, self.z1 = z0, z1
        self.nl = z1 - z0
        self.h, self.tol = h, tol
        self.phi = np.full((self.nl + 2, ny, nx), INF)  # ghost planes at 0 and nl+1
        self.speed = np.asarray(speed, dtype=np.float64)[z0:z1].copy()
        self.state = np.asarray(state, dtype=np.uint8)[z0:z1].copy()
        self.label = np.zeros((self.nl, ny, nx), dtype=np.uint8)
        self.active = []  # local (z, y, x) of owned cells
        self.member = None
        self.D = np.zeros((self.nl, ny, nx), dtype=bool)

    # ---- helpers -------------------------------------------------------
    def _vals(self, snap, cells):
        if not cells:
            return np.zeros(0)
        z = np.array([c[0] for c in cells]) + 1
        y = np.array([c[1] for c in cells])
        x = np.array([c[2] for c in cells])
        P = np.pad(snap, ((0, 0), (1, 1), (1, 1)), constant_values=INF)  # +inf x/y border
        xm = np.minimum(P[z, y + 1, x], P[z, y + 1, x + 2])
        ym = np.minimum(P[z, y, x + 1], P[z, y + 2, x + 1])
        zm = np.minimum(P[z - 1, y + 1, x + 1], P[z + 1, y + 1, x + 1])
        f = self.speed[z - 1, y, x]
        return cpu.local_3d_uniform(xm, ym, zm, f, self.h)

    def _nbrs(self, z, y, x):
        # reference order W, E, S, N, D, U (E/ifim.py:35-45 plus z); z may be -1 / nl (ghost)
        if x > 0:
            yield z, y, x - 1
        if x < self.nx - 1:
            yield z, y, x + 1
        if y > 0:
            yield z, y - 1, x
        if y < self.ny - 1:
            yield z, y + 1, x
        if self.z0 + z > 0:
            yield z - 1, y, x
        if self.z0 + z < self.nz - 1:
            yield z + 1, y, x

    def _owned(self, z):
        return 0 <= z < self.nl

    # ---- SlabEngine ----------------------------------------------------
    def boundary_planes(self):
        return torch.from_numpy(self.phi[1].copy()), torch.from_numpy(self.phi[self.nl].copy())

    def set_ghosts(self, lo, hi):
        self.phi[0] = INF if lo is None else lo.numpy()
        self.phi[self.nl + 1] = INF if hi is None else hi.numpy()

    def init_active(self, seeds):
        nx, ny = self.nx, self.ny
        gl = []
        for c, v in seeds:
            z, r = divmod(c, nx * ny)
            y, x = divmod(r, nx)
            gl.append((z, y, x))
            if self.z0 <= z < self.z1:
                self.phi[z - self.z0 + 1, y, x] = v
                self.state[z - self.z0, y, x] = SOURCE
        for (gz, y, x) in gl:  # E/ifim.py:97-102 over every seed, owned neighbours only
            for (nz_, ny_, nx_) in self._nbrs(gz - self.z0, y, x):
                if not self._owned(nz_):
                    continue
                st = self.state[nz_, ny_, nx_]
                if st != BLOCKED and st != SOURCE and self.label[nz_, ny_, nx_] == FAR:
                    self.label[nz_, ny_, nx_] = ACTIVE
                    self.active.append((nz_, ny_, nx_))
        return len(self.active)

    def update_local(self):
        snap = self.phi.copy()
        vals = self._vals(snap, self.active)
        req_lo = np.zeros((self.ny, self.nx), dtype=np.uint8)
        req_hi = np.zeros((self.ny, self.nx), dtype=np.uint8)
        surv = []
        for (z, y, x), v in zip(self.active, vals.tolist()):
            old = snap[z + 1, y, x]
            if v == old or abs(v - old) <= self.tol:
                self.label[z, y, x] = CONVERGED
                for (nz_, ny_, nx_) in self._nbrs(z, y, x):
                    if snap[nz_ + 1, ny_, nx_] != INF:
                        continue
                    if nz_ < 0:
                        req_lo[ny_, nx_] = 1
                    elif nz_ >= self.nl:
                        req_hi[ny_, nx_] = 1
                    elif self.state[nz_, ny_, nx_] != BLOCKED and self.label[nz_, ny_, nx_] == FAR:
                        self.label[nz_, ny_, nx_] = ACTIVE
                        surv.append((nz_, ny_, nx_))
            else:
                self.phi[z + 1, y, x] = v
                surv.append((z, y, x))
        self.active = surv
        return torch.from_numpy(req_lo), torch.from_numpy(req_hi)

    def apply_requests(self, from_lo, from_hi):
        for plane, z in ((from_lo, 0), (from_hi, self.nl - 1)):
            if plane is None:
                continue
            for y, x in zip(*np.nonzero(plane.numpy())):
                if self.state[z, y, x] != BLOCKED and self.label[z, y, x] == FAR:
                    self.label[z, y, x] = ACTIVE
                    self.active.append((z, int(y), int(x)))
        return len(self.active)

    def build_local(self):
        free = (self.state != BLOCKED) & (self.state != SOURCE)
        cells = [tuple(c) for c in np.argwhere(free)]
        vals = self._vals(self.phi.copy(), cells)
        self.member = np.zeros_like(free)
        with np.errstate(invalid="ignore"):
            for (z, y, x), v in zip(cells, vals.tolist()):
                if abs(v - self.phi[z + 1, y, x]) > self.tol:
                    self.member[z, y, x] = True
        return len(cells), int(self.member.sum())

    def remedy_boundary_d(self):
        return (torch.from_numpy(self.D[0].astype(np.uint8)), torch.from_numpy(self.D[-1].astype(np.uint8)))

    def remedy_local(self, g_lo, g_hi, first):
        free = (self.state != BLOCKED) & (self.state != SOURCE)
        if first:
            R = self.member
        else:
            Dg = np.zeros((self.nl + 2, self.ny, self.nx), dtype=bool)
            Dg[1:-1] = self.D
            if g_lo is not None:
                Dg[0] = g_lo.numpy().astype(bool)
            if g_hi is not None:
                Dg[-1] = g_hi.numpy().astype(bool)
            dil = np.zeros_like(self.D)
            dil[:, :, 1:] |= self.D[:, :, :-1]
            dil[:, :, :-1] |= self.D[:, :, 1:]
            dil[:, 1:, :] |= self.D[:, :-1, :]
            dil[:, :-1, :] |= self.D[:, 1:, :]
            dil |= Dg[:-2] | Dg[2:]
            R = self.D | (dil & free)
        cells = [tuple(c) for c in np.argwhere(R)]
        snap = self.phi.copy()
        vals = self._vals(snap, cells)
        D = np.zeros_like(self.D)
        for (z, y, x), v in zip(cells, vals.tolist()):
            if v < snap[z + 1, y, x] - self.tol:
                self.phi[z + 1, y, x] = v
                D[z, y, x] = True
        self.D = D
        return len(cells), int(D.sum())

    def result(self):
        return self.phi[1:-1].copy()
