mkdir -p gpurun_out
timeout 300 tools/cuda/check_sqrt 8 > gpurun_out/r5_check_sqrt.log 2>&1; echo "check_sqrt rc=$?"; cat gpurun_out/r5_check_sqrt.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_brick.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r5_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r5_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_base.so libeik_ifim.so libeik_base.so:EIK_REMEDY=brick libeik_ifim.so:EIK_REMEDY=brick > gpurun_out/r5_ab_cfg4.log 2>&1; cat gpurun_out/r5_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_base.so:EIK_REMEDY=list libeik_ifim.so:EIK_REMEDY=list libeik_base.so:EIK_REMEDY=brick libeik_ifim.so:EIK_REMEDY=brick > gpurun_out/r5_ab_cfg5.log 2>&1; cat gpurun_out/r5_ab_cfg5.log
