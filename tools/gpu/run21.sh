mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fixpoint.py -q -p no:cacheprovider -k "bench" > gpurun_out/r21_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r21_tests.log
