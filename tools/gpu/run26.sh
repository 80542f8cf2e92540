mkdir -p gpurun_out
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_mu2.so libeik_mu2b2.so > gpurun_out/r26_ab_cfg4.log 2>&1; cat gpurun_out/r26_ab_cfg4.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_ifim.so libeik_mu2.so libeik_mu2b2.so > gpurun_out/r26_ab_cfg3.log 2>&1; cat gpurun_out/r26_ab_cfg3.log
