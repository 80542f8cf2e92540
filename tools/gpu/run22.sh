mkdir -p gpurun_out
for c in 0 16 32 64 96; do
EIK_UPD_CTAS=$c python - <<'PY' >> gpurun_out/r22_ctas.log 2>&1
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench, paper_2106_15869_b200 as eik
dev = torch.device("cuda:0")
for cfg, n in (("cfg2", 4096), ("cfg1", 256), ("cfg3", 256)):
    w = bench.make_workload(torch, dev, cfg, n)
    best = None
    for _ in range(5):
        g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device=dev), w.F, torch.zeros(w.shape, dtype=torch.uint8, device=dev))
        r = eik.solve_ifim(g, w.bc(eik)); torch.cuda.synchronize()
        d = r.stats.device_ms
        best = d if best is None or d["update"] < best["update"] else best
    print("ctas", os.environ["EIK_UPD_CTAS"], cfg, "update ms", round(best["update"], 3), "total", round(best["total"], 3), r.stats.solver_calls)
PY
done
cat gpurun_out/r22_ctas.log
