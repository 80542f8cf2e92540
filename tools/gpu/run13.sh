mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_slab_peer_gpu.py -x -q -p no:cacheprovider > gpurun_out/r13_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r13_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_upf0.so libeik_ifim.so > gpurun_out/r13_ab_cfg4.log 2>&1; cat gpurun_out/r13_ab_cfg4.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_upf0.so libeik_ifim.so > gpurun_out/r13_ab_cfg3.log 2>&1; cat gpurun_out/r13_ab_cfg3.log
for so in libeik_upf0.so libeik_ifim.so; do python - "$so" <<'PY' >> gpurun_out/r13_cfg2.log 2>&1
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2106_15869_b200 import _native
_native.LIB = os.path.join(os.path.dirname(_native.LIB), sys.argv[1])
import torch, bench, paper_2106_15869_b200 as eik
dev = torch.device("cuda:0")
for cfg, n in (("cfg2", 4096), ("cfg1", 256)):
    w = bench.make_workload(torch, dev, cfg, n)
    best = None
    for _ in range(5):
        g = w.grid(eik, torch.full(w.shape, float("inf"), dtype=torch.float64, device=dev), w.F, torch.zeros(w.shape, dtype=torch.uint8, device=dev))
        r = eik.solve_ifim(g, w.bc(eik)); torch.cuda.synchronize()
        d = r.stats.device_ms
        best = d if best is None or d["total"] < best["total"] else best
    print(sys.argv[1], cfg, {k: round(v, 3) for k, v in best.items()}, r.stats.solver_calls)
PY
done; cat gpurun_out/r13_cfg2.log
