mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py -q -p no:cacheprovider --durations=5 > gpurun_out/r40_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r40_tests.log
