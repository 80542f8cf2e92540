mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_brick.py -x -q -p no:cacheprovider > gpurun_out/r25_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r25_tests.log
timeout 900 python tools/fuzz_brick.py 600 31 > gpurun_out/r25_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/r25_fuzz.log
export EIK_REMEDY=brick
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_fill0.so libeik_ifim.so > gpurun_out/r25_ab_cfg5.log 2>&1; cat gpurun_out/r25_ab_cfg5.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_fill0.so libeik_ifim.so > gpurun_out/r25_ab_cfg4.log 2>&1; cat gpurun_out/r25_ab_cfg4.log
