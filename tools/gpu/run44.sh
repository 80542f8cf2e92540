mkdir -p gpurun_out
timeout 1500 python tools/ab.py --n 1024 --kind cfg5 libeik_ifim.so libeik_mu2.so libeik_mu2b2.so > gpurun_out/r44_ab.log 2>&1; cat gpurun_out/r44_ab.log
