mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fixpoint.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "pinned or bench_json or pinned_host or host" > gpurun_out/r31_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r31_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err; echo "bench rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/r31_bench.json').read().strip().splitlines()[-1]); print('device ms', round(d['ms_per_step'],1), 'e2e', d['e2e'], d['parity'])"
