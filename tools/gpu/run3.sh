mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_brick.py -x -q -p no:cacheprovider > gpurun_out/r3_brick_tests.log 2>&1; echo "brick tests rc=$?"; tail -3 gpurun_out/r3_brick_tests.log
export EIK_REMEDY=brick
timeout 900 python tools/ab.py --n 512 --kind checker libeik_bal0.so libeik_bal1s0.so libeik_ifim.so libeik_ifim.so:EIK_REMEDY=list > gpurun_out/r3_ab_cfg4.log 2>&1; cat gpurun_out/r3_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_bal0.so libeik_bal1s0.so libeik_ifim.so > gpurun_out/r3_ab_cfg5.log 2>&1; cat gpurun_out/r3_ab_cfg5.log
