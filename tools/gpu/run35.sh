export EIK_REMEDY=list
timeout 900 python tools/ab.py --n 512 --kind checker libeik_l1pf0.so libeik_ifim.so > gpurun_out/r35_ab_cfg4.log 2>&1; cat gpurun_out/r35_ab_cfg4.log
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_l1pf0.so libeik_ifim.so > gpurun_out/r35_ab_cfg5.log 2>&1; cat gpurun_out/r35_ab_cfg5.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_l1pf0.so libeik_ifim.so > gpurun_out/r35_ab_cfg3.log 2>&1; cat gpurun_out/r35_ab_cfg3.log
