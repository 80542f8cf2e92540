mkdir -p gpurun_out
timeout 1500 python tools/fuzz_peer.py 600 19 > gpurun_out/r47_fuzz_peer.log 2>&1; echo "peer rc=$?"; tail -2 gpurun_out/r47_fuzz_peer.log
timeout 1500 python tools/fuzz_brick.py 1500 47 > gpurun_out/r47_fuzz_brick.log 2>&1; echo "brick rc=$?"; tail -1 gpurun_out/r47_fuzz_brick.log
timeout 1500 python tools/fuzz_parity.py 2000 53 > gpurun_out/r47_fuzz_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r47_fuzz_parity.log
