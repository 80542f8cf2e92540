mkdir -p gpurun_out
timeout 1500 python tools/fuzz_brick.py 1500 11 > gpurun_out/r24_fuzz_brick.log 2>&1; echo "fuzz brick rc=$?"; tail -3 gpurun_out/r24_fuzz_brick.log
timeout 1200 python tools/fuzz_parity.py 1500 23 > gpurun_out/r24_fuzz_parity.log 2>&1; echo "fuzz parity rc=$?"; tail -3 gpurun_out/r24_fuzz_parity.log
