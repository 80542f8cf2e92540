mkdir -p gpurun_out
export EIK_REMEDY=list
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/r8_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r8_tests.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_mlpf0.so libeik_mlpf1.so > gpurun_out/r8_ab_cfg4.log 2>&1; cat gpurun_out/r8_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_mlpf0.so libeik_mlpf1.so > gpurun_out/r8_ab_cfg5.log 2>&1; cat gpurun_out/r8_ab_cfg5.log
