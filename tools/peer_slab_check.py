"""torchrun check of the distributed peer-slab path (torch symmetric memory):
every rank solves its slab of a small 3D problem through DistributedSlabs; the
gathered field and stats must equal the single-device solve bit for bit.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/peer_slab_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2106_15869_b200 as eik  # noqa: E402
from paper_2106_15869_b200.slab import SlabPartition  # noqa: E402
from paper_2106_15869_b200.slab_peer import DistributedSlabs  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    nz, ny, nx = 40, 24, 36
    kk, jj, ii = np.mgrid[0:nz, 0:ny, 0:nx]
    F = torch.as_tensor(np.where(((ii // 4) + (jj // 4) + (kk // 4)) % 2 == 0, 1.0, 0.01), device=dev)
    seeds = [((5 * ny + 7) * nx + 3, 0.0), ((33 * ny + 20) * nx + 30, 0.5)]
    z0, z1 = SlabPartition(nz, world).bounds(rank)
    ds = DistributedSlabs((nz, ny, nx), 0.5)
    st = torch.zeros((z1 - z0, ny, nx), dtype=torch.uint8, device=dev)
    ok = True
    for rep in range(2):  # reuse of the symmetric buffers
        st.zero_()
        phi, s = ds.solve(F[z0:z1].contiguous(), st, seeds)
        parts = [torch.empty(0)] * world
        dist.all_gather_object(parts, phi.cpu())
        if rank == 0:
            g = eik.Grid3D(nx, ny, nz, 0.5, (0.0, 0.0, 0.0),
                           torch.full((nz, ny, nx), float("inf"), dtype=torch.float64, device=dev), F,
                           torch.zeros((nz, ny, nx), dtype=torch.uint8, device=dev))
            ref = eik.solve_ifim(g, eik.BoundaryCondition(tuple((eik.CellIndex3D(c % nx, (c // nx) % ny, c // (nx * ny)), v)
                                                                for c, v in seeds)))
            got = torch.cat(parts, 0)
            same = torch.equal(got, ref.phi.cpu()) and s.solver_calls == ref.stats.solver_calls and \
                s.active_history == ref.stats.active_history and s.peak_remedy == ref.stats.peak_remedy
            print(f"rep {rep}: world {world} bit-identical={same} calls={s.solver_calls}", flush=True)
            ok &= same
    flag = torch.tensor([int(ok)], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    return 0 if flag.item() else 1


if __name__ == "__main__":
    sys.exit(main())
