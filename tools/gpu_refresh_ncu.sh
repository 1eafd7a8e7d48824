set -x
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
ncu --set full --clock-control none -k regex:"refresh" --launch-skip 9 -c 3 -o gpurun_out/refresh -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/refresh_bench.log 2>&1
echo ncu $?
FT_REFRESH=simt ncu --set full --clock-control none -k regex:"refresh" --launch-skip 9 -c 3 -o gpurun_out/refresh_simt -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/refresh_bench2.log 2>&1
echo ncu2 $?
