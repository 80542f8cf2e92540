mkdir -p gpurun_out
export EIK_REMEDY=list
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r43_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r43_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_lc0.so libeik_ifim.so > gpurun_out/r43_ab.log 2>&1; cat gpurun_out/r43_ab.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_lc0.so libeik_ifim.so >> gpurun_out/r43_ab.log 2>&1; tail -2 gpurun_out/r43_ab.log
