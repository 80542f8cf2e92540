mkdir -p gpurun_out
export EIK_REMEDY=brick
timeout 600 python -m pytest tests/test_gpu_brick.py -x -q -p no:cacheprovider > gpurun_out/r4_brick_tests.log 2>&1; echo "brick tests rc=$?"; tail -2 gpurun_out/r4_brick_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_bal0.so libeik_ifim.so libeik_sus1k.so libeik_sus100k.so > gpurun_out/r4_ab_cfg4.log 2>&1; cat gpurun_out/r4_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_bal0.so libeik_ifim.so libeik_sus1k.so > gpurun_out/r4_ab_cfg5.log 2>&1; cat gpurun_out/r4_ab_cfg5.log
