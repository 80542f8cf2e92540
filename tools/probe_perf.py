"""Quick device-time probe of the BASELINE configs (not the bench; no clocks/roofline)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_15869_b200 as eik

def checker(n, blk):
    k = torch.arange(n, device="cuda") // blk
    return torch.where(((k[None, None, :] + k[None, :, None] + k[:, None, None]) % 2) == 0, torch.tensor(1.0, dtype=torch.float64), torch.tensor(0.01, dtype=torch.float64))

def run(name, n, F, seeds, reps=2):
    dev = torch.device("cuda:0")
    for r in range(reps):
        phi = torch.full((n, n, n), float("inf"), dtype=torch.float64, device=dev)
        state = torch.where(F == 0, 4, 0).to(torch.uint8)
        g = eik.Grid3D(n, n, n, 1.0, (0.0, 0.0, 0.0), phi, F, state)
        bc = eik.BoundaryCondition(tuple((eik.CellIndex3D(*s), 0.0) for s in seeds))
        torch.cuda.synchronize(); t = time.perf_counter()
        res = eik.solve_ifim(g, bc)
        torch.cuda.synchronize(); t = time.perf_counter() - t
        s = res.stats
        print(f"{name} rep{r}: wall {t*1e3:.1f} ms dev {s.device_ms} calls {s.solver_calls} it {s.iterations} "
              f"phases {s.phases} peakA {s.peak_active} peakR {s.peak_remedy} writes {s.phi_writes} "
              f"-> {s.solver_calls/ (s.device_ms['total']/1e3):.3e} upd/s", flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
run(f"checker{n}", n, checker(n, n // 16), [(n // 2, n // 2, n // 2)])
rng = np.random.default_rng(2106)
seeds = [tuple(int(v) for v in rng.integers(0, n, 3)) for _ in range(16)]
run(f"const16_{n}", n, torch.ones((n, n, n), dtype=torch.float64, device="cuda"), seeds)
