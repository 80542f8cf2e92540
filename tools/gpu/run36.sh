mkdir -p gpurun_out
timeout 1200 python tools/make_gpu_crosscheck.py 1024 > gpurun_out/r36_crosscheck.log 2>&1; echo "crosscheck rc=$?"; tail -5 gpurun_out/r36_crosscheck.log
mkdir -p gpurun_out/golden; cp tests/golden/fullsize_gpu.json gpurun_out/golden/ 2>/dev/null
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/r36_bench_cfg5.json 2> gpurun_out/r36_bench_cfg5.err; echo "bench rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/r36_bench_cfg5.json').read().strip().splitlines()[-1]); print(d['parity'], d['parity_detail'], d['roofline'])"
