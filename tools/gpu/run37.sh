mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/r37_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r37_tests.log
