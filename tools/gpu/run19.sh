mkdir -p gpurun_out
for eng in auto list brick; do
  EIK_REMEDY=$eng timeout 600 python bench.py --config cfg5 --dtype f32 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r19_cfg5_f32_$eng.json 2> gpurun_out/r19_cfg5_f32_$eng.err; echo "cfg5 f32 $eng rc=$?"
  EIK_REMEDY=$eng timeout 600 python bench.py --config cfg4 --dtype f32 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r19_cfg4_f32_$eng.json 2> gpurun_out/r19_cfg4_f32_$eng.err; echo "cfg4 f32 $eng rc=$?"
done
timeout 600 python -m pytest tests/test_gpu_f32.py -x -q -p no:cacheprovider > gpurun_out/r19_f32_tests.log 2>&1; echo "f32 tests rc=$?"; tail -2 gpurun_out/r19_f32_tests.log
