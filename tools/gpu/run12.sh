mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r12_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r12_gputest.log
python __graft_entry__.py smoke > gpurun_out/r12_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r12_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r12_bench.json 2> gpurun_out/r12_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/r12_bench_cfg5.json 2> gpurun_out/r12_bench_cfg5.err; echo "bench cfg5 rc=$?"
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/r12_bench_cfg3.json 2> gpurun_out/r12_bench_cfg3.err; echo "bench cfg3 rc=$?"
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 > gpurun_out/r12_bench_cfg2.json 2> gpurun_out/r12_bench_cfg2.err; echo "bench cfg2 rc=$?"
