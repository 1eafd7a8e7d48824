# quadw per-step lookahead (FT_QUADW_LA 0/1/2) vs the Gram form on the row shards of Netflix
# mode 2 and order-4 (tools/time_shards.py), plus the quadw parity cases
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py -q -m gpu -k "quadw or without_fibers" > gpurun_out/pytest_quadw.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_quadw.log
for cfg in "0 0" "0 1" "0 2" "1 1"; do
  set -- $cfg
  FT_QUADW_GRAM=$1 FT_QUADW_LA=$2 timeout 600 python tools/time_shards.py netflix32 --modes 2 --P 1 2 4 8 > gpurun_out/sh_nf_g$1_la$2.json 2> gpurun_out/sh_nf_g$1_la$2.err; echo nf $1 $2 $?
  grep netflix32 gpurun_out/sh_nf_g$1_la$2.err
done
for cfg in "0 0" "0 2" "1 1"; do
  set -- $cfg
  FT_QUADW_GRAM=$1 FT_QUADW_LA=$2 timeout 900 python tools/time_shards.py order4 --modes 0 --P 4 8 > gpurun_out/sh_o4_g$1_la$2.json 2> gpurun_out/sh_o4_g$1_la$2.err; echo o4 $1 $2 $?
  grep order4 gpurun_out/sh_o4_g$1_la$2.err
done
