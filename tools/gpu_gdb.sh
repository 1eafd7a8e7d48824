# Gram form double-buffered (FT_QUADW_DB) on the row shards + parity
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py tests/test_netflix_parity_gpu.py -q -m gpu -x -k "quadw or long_rows" > gpurun_out/pytest_gdb.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_gdb.log
for db in 1 0; do
FT_QUADW_DB=$db timeout 600 python tools/time_shards.py netflix32 --P 1 2 4 8 > gpurun_out/gdb_$db.json 2> gpurun_out/gdb_$db.err; echo sh $db $?
grep netflix32 gpurun_out/gdb_$db.err
done
timeout 600 python bench.py --no-cpu --no-ncu > gpurun_out/gdb_bench.json 2> gpurun_out/gdb_bench.err; echo bench $?
python -c "
import json; d=json.load(open('gpurun_out/gdb_bench.json'))
print('bench', d['value']/1e9, d['e2e']['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
