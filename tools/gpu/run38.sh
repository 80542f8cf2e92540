export EIK_REMEDY=list
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_mu3b3.so libeik_mu4b2.so libeik_mu3b4.so > gpurun_out/r38_ab_cfg4.log 2>&1; cat gpurun_out/r38_ab_cfg4.log
