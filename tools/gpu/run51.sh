# final round-2 evidence after the staged 3D expansion: GPU suite, smoke, bench (cfg4 both arms, cfg3, cfg2),
# usage: P=<prefix> bash tools/gpu/run51.sh
# launch list, ncu --set full of the list remedy kernel on cfg4
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${P:-i}_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/${P:-i}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${P:-i}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${P:-i}_smoke.log
python bench.py > gpurun_out/${P:-i}_bench.log 2> gpurun_out/${P:-i}_bench.err
python bench.py --config cfg3 > gpurun_out/${P:-i}_cfg3.log 2> gpurun_out/${P:-i}_cfg3.err
python bench.py --config cfg2 > gpurun_out/${P:-i}_cfg2.log 2> gpurun_out/${P:-i}_cfg2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P:-i}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/${P:-i}_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_remedy$" -s 1 -c 1 -o gpurun_out/${P:-i}_prof_list_cfg4 python tools/prof_solve.py cfg4 512 2 > gpurun_out/${P:-i}_ncu.log 2>&1
echo done > gpurun_out/${P:-i}_done
