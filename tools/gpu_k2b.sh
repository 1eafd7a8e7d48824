# K2 TMA form: full GPU suite, bench, K2 timing, ncu of the refresh launches
set -x
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/k2b_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/k2b_pytest.log
timeout 900 python bench.py > gpurun_out/k2b_bench.json 2> gpurun_out/k2b_bench.err; echo bench $?
timeout 300 python tools/time_refresh.py > gpurun_out/k2b_time.log 2>&1; echo time $?
cat gpurun_out/k2b_time.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"refresh_t" --launch-skip 6 -c 3 \
  -o gpurun_out/k2b_refresh -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/k2b_refresh.log 2>&1
echo refresh $?
