mkdir -p gpurun_out
export EIK_REMEDY=brick
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_ifim.so libeik_dt0c3.so libeik_dt0c2.so libeik_dt0c3u1.so libeik_dt1c2u1.so > gpurun_out/r9_ab_cfg5.log 2>&1; cat gpurun_out/r9_ab_cfg5.log
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_dt0c3.so libeik_dt0c2.so libeik_dt0c3u1.so > gpurun_out/r9_ab_cfg4.log 2>&1; cat gpurun_out/r9_ab_cfg4.log
