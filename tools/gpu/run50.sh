# final round-2 evidence with the 512-thread remedy CTAs: GPU suite, bench (both arms), launch list,
# ncu --set full of the list remedy kernel on cfg4
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/f_gputest.log
python bench.py > gpurun_out/f_bench.log 2> gpurun_out/f_bench.err
python bench.py --impl reference > gpurun_out/f_ref.log 2> gpurun_out/f_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/f_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_remedy<' -s 1 -c 1 -o gpurun_out/f_prof_list_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/f_ncu.log 2>&1
echo done > gpurun_out/f_done
