mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fixpoint.py -x -q -p no:cacheprovider -k "pinned or bench_json" > gpurun_out/r28_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r28_tests.log
for i in 1 2; do timeout 900 python bench.py --no-cpu > gpurun_out/r28_bench_$i.json 2> gpurun_out/r28_bench_$i.err; echo "bench rc=$?"; python -c "
import json
d=json.loads(open('gpurun_out/r28_bench_$i.json').read().strip().splitlines()[-1]); print('device ms', round(d['ms_per_step'],1), 'e2e', d['e2e'])"; done
