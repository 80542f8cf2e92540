mkdir -p gpurun_out
python tools/prof_solve.py cfg5 1024 1 > gpurun_out/r17_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_remedy_b -c 1 -o gpurun_out/prof_brick_cfg5_1024 python tools/prof_solve.py cfg5 1024 1 > gpurun_out/r17_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r17_plain.log
