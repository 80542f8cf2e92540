mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r23_gputest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r23_gputest.log
python __graft_entry__.py smoke > gpurun_out/r23_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r23_smoke.log
timeout 900 python bench.py > gpurun_out/r23_bench.json 2> gpurun_out/r23_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r23_bench.json
