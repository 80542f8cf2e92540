mkdir -p gpurun_out
timeout 900 python tools/ab.py --n 512 --kind checker libeik_ifim.so libeik_spin0.so libeik_spin8.so libeik_spin128.so > gpurun_out/r11_ab_cfg4.log 2>&1; cat gpurun_out/r11_ab_cfg4.log
timeout 900 python tools/ab.py --n 256 --kind const libeik_ifim.so libeik_spin0.so libeik_spin8.so libeik_spin128.so > gpurun_out/r11_ab_cfg3.log 2>&1; cat gpurun_out/r11_ab_cfg3.log
