mkdir -p gpurun_out
set -x
export EIK_REMEDY=brick
python tools/prof_solve.py cfg5 512 2 > gpurun_out/p2_plain_b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_remedy_b -s 1 -c 1 -o gpurun_out/prof_brick_cfg5 python tools/prof_solve.py cfg5 512 2 > gpurun_out/p2_ncu_b.log 2>&1
echo "ncu brick rc=$?"
python tools/prof_solve.py cfg4 512 2 > gpurun_out/p2_plain_b4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_remedy_b -s 1 -c 1 -o gpurun_out/prof_brick_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/p2_ncu_b4.log 2>&1
echo "ncu brick4 rc=$?"
export EIK_REMEDY=list
python tools/prof_solve.py cfg4 512 2 > gpurun_out/p2_plain_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_remedy<' -s 1 -c 1 -o gpurun_out/prof_list_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/p2_ncu_l.log 2>&1
echo "ncu list rc=$?"
