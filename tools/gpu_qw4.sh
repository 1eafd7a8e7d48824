set -x
timeout 1800 python -m pytest tests -q -m gpu -x -k "quad_sweeps or netflix or quadw or variant" > gpurun_out/qw4_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/qw4_pytest.log
timeout 1200 python tools/time_shards.py order4 --P 1 2 4 8 --modes 0 > gpurun_out/qw4_o4.json 2> gpurun_out/qw4_o4.err; echo o4 $?
tail -4 gpurun_out/qw4_o4.err
FT_QUADW_GRAM=1 timeout 1200 python tools/time_shards.py order4 --P 4 8 --modes 0 > /dev/null 2> gpurun_out/qw4_o4g.err; echo o4g $?
tail -2 gpurun_out/qw4_o4g.err
timeout 900 python tools/time_shards.py netflix32 > gpurun_out/qw4_nf.json 2> gpurun_out/qw4_nf.err; echo nf $?
tail -4 gpurun_out/qw4_nf.err
