mkdir -p gpurun_out
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_sn1.so libeik_ifim.so:EIK_REMEDY=brick libeik_sn1.so:EIK_REMEDY=brick > gpurun_out/r6_ab_cfg4.log 2>&1; cat gpurun_out/r6_ab_cfg4.log
