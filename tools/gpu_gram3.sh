set -x
timeout 900 python tools/time_shards.py netflix32 --P 4 8 --modes 2 > gpurun_out/gram3_shards.json 2> gpurun_out/gram3_shards.err; echo shards $?
tail -3 gpurun_out/gram3_shards.err
timeout 1500 python -m pytest tests -q -m gpu -x -k "quad_sweeps or netflix or quadw" > gpurun_out/gram3_pytest.log 2>&1; echo pytest $?
tail -1 gpurun_out/gram3_pytest.log
