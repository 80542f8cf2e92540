set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/gputest.log
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
for eng in auto list brick; do
  EIK_REMEDY=$eng timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_cfg4_$eng.json 2> gpurun_out/bench_cfg4_$eng.err; echo "cfg4 $eng rc=$?"
done
for eng in auto list; do
  EIK_REMEDY=$eng timeout 900 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg5_$eng.json 2> gpurun_out/bench_cfg5_$eng.err; echo "cfg5 $eng rc=$?"
done
