# quadw producers with pipelined gathers: parity + row-shard timings + bench
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py tests/test_netflix_parity_gpu.py -q -m gpu -x -k "quadw or long_rows or without_fibers" > gpurun_out/pytest_pipe.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_pipe.log
for g in 0 1; do
  FT_QUADW_GRAM=$g timeout 600 python tools/time_shards.py netflix32 --modes 2 --P 1 4 8 > gpurun_out/shp_nf_g$g.json 2> gpurun_out/shp_nf_g$g.err; echo nf $g $?
  grep netflix32 gpurun_out/shp_nf_g$g.err
  FT_QUADW_GRAM=$g timeout 900 python tools/time_shards.py order4 --modes 0 --P 8 > gpurun_out/shp_o4_g$g.json 2> gpurun_out/shp_o4_g$g.err; echo o4 $g $?
  grep order4 gpurun_out/shp_o4_g$g.err
done
timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/pipe_bench.json 2> gpurun_out/pipe_bench.err; echo bench $?
python -c "
import json; d=json.load(open('gpurun_out/pipe_bench.json'))
print('bench', d['value']/1e9, d['factor_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
