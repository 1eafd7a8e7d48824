# ncu --set full of one kernel launch: $1 = kernel regex, $2 = launch-skip, $3 = env assignments
set -x
env $3 ncu --set full --clock-control none --import-source on -k regex:"$1" --launch-skip $2 -c 1 \
  -o gpurun_out/one -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/one.log 2>&1
echo ncu $?
tail -3 gpurun_out/one.log
