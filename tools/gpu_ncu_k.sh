# ncu --set full of one launch of kernel regex $1 after skipping $2 matching launches
set -x
ncu --set full --clock-control none --import-source on -k regex:"$1" --launch-skip $2 -c 1 \
  -o gpurun_out/k_one -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/k_one.log 2>&1
echo ncu $?
