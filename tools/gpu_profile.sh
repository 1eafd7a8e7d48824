# ncu evidence for the current kernels (run under gpurun; outputs in gpurun_out/)
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
echo launches $?
# one timed epoch's six sweeps (warm-up 3 epochs = 9 factor + 9 core launches skipped)
ncu --set full --clock-control none --import-source on -k regex:"factor_rows|core_rows" \
  --launch-skip 18 -c 6 -o gpurun_out/sweeps -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweeps_bench.log 2>&1
echo sweeps $?
