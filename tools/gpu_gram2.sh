# quadw Gram form v2: parity (quad cases incl. forced forms, Netflix-scale), shard times, ncu at P = 8
set -x
timeout 1500 python -m pytest tests -q -m gpu -x -k "quad_sweeps or netflix or quadw" > gpurun_out/gram2_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/gram2_pytest.log
timeout 900 python tools/time_shards.py netflix32 > gpurun_out/gram2_shards.json 2> gpurun_out/gram2_shards.err; echo shards $?
tail -4 gpurun_out/gram2_shards.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qw2_p8 -f \
  python tools/time_shards.py netflix32 --P 8 --modes 2 --reps 1 > gpurun_out/qw2_p8.log 2>&1; echo p8 $?
