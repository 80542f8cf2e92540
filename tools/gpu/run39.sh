mkdir -p gpurun_out
export EIK_REMEDY=list
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/r39_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r39_tests.log
timeout 900 python tools/fuzz_parity.py 400 77 > gpurun_out/r39_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/r39_fuzz.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_dza0.so libeik_ifim.so > gpurun_out/r39_ab_cfg4.log 2>&1; cat gpurun_out/r39_ab_cfg4.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_dza0.so libeik_ifim.so > gpurun_out/r39_ab_cfg3.log 2>&1; cat gpurun_out/r39_ab_cfg3.log
