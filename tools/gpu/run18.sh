mkdir -p gpurun_out
export EIK_REMEDY=list
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_to1.so libeik_to2.so > gpurun_out/r18_ab_cfg4.log 2>&1; cat gpurun_out/r18_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_ifim.so libeik_to1.so libeik_to2.so > gpurun_out/r18_ab_cfg5.log 2>&1; cat gpurun_out/r18_ab_cfg5.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_ifim.so libeik_to1.so libeik_to2.so > gpurun_out/r18_ab_cfg3.log 2>&1; cat gpurun_out/r18_ab_cfg3.log
