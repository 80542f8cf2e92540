mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r16_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r16_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_lazy0.so libeik_ifim.so libeik_lazy0.so:EIK_REMEDY=brick libeik_ifim.so:EIK_REMEDY=brick > gpurun_out/r16_ab_cfg4.log 2>&1; cat gpurun_out/r16_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_lazy0.so libeik_ifim.so > gpurun_out/r16_ab_cfg5.log 2>&1; cat gpurun_out/r16_ab_cfg5.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_lazy0.so libeik_ifim.so > gpurun_out/r16_ab_cfg3.log 2>&1; cat gpurun_out/r16_ab_cfg3.log
