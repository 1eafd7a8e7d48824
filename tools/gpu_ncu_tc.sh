# ncu --set full of one tcgen05 factor launch (mode 0 of the 3rd warm-up epoch) + one quadr launch
set -x
ncu --set full --clock-control none --import-source on -k regex:"factor_rows_tc" --launch-skip 4 -c 1 \
  -o gpurun_out/tc_one -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/tc_one.log 2>&1
echo ncu $?
tail -3 gpurun_out/tc_one.log
