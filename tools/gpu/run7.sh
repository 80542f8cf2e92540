mkdir -p gpurun_out
export EIK_REMEDY=brick
timeout 900 python tools/ab.py --n 512 --kind cfg5 libeik_ifim.so libeik_n1c3.so libeik_n1c2.so libeik_n3c1.so > gpurun_out/r7_ab_brick.log 2>&1; cat gpurun_out/r7_ab_brick.log
unset EIK_REMEDY
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r7_bench_plain.json 2> gpurun_out/r7_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r7_ncu_launch.log 2>&1
echo "launch list rc=$?"
export EIK_REMEDY=list
python tools/prof_solve.py cfg4 512 2 > gpurun_out/r7_plain_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_remedy -s 1 -c 1 -o gpurun_out/prof_list_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/r7_ncu_l.log 2>&1
echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_update -s 1 -c 1 -o gpurun_out/prof_update_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/r7_ncu_u.log 2>&1
echo "ncu update rc=$?"
