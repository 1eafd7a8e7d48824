# K2 streaming refresh: parity tests, event timing, ncu of the three Netflix refreshes
set -x
timeout 600 python -m pytest tests -q -m gpu -k "refresh or config1 or peer" > gpurun_out/k2_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/k2_pytest.log
timeout 300 python tools/time_refresh.py > gpurun_out/k2_time.log 2>&1; echo time $?
cat gpurun_out/k2_time.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"refresh_t" --launch-skip 6 -c 3 \
  -o gpurun_out/k2_refresh -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/k2_refresh.log 2>&1
echo refresh $?
