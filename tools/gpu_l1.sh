# quadw double-buffered per-step form (FT_QUADW_DB) A/B + K4 direct with minimal shared memory
set -x
timeout 1200 python -m pytest tests/test_quad_gpu.py tests/test_gpu_parity.py tests/test_netflix_parity_gpu.py -q -m gpu -x > gpurun_out/pytest_l1.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_l1.log
for db in 1 0; do
FT_QUADW_DB=$db timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/l1_$db.json 2> gpurun_out/l1_$db.err; echo bench db=$db $?
python -c "
import json; d=json.load(open('gpurun_out/l1_$db.json'))
print('db=$db', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()}, d['train_rmse'])"
FT_QUADW_GRAM=0 FT_QUADW_DB=$db timeout 600 python tools/time_shards.py netflix32 --modes 2 --P 4 8 > gpurun_out/l1sh_$db.json 2> gpurun_out/l1sh_$db.err; echo sh $db $?
grep netflix32 gpurun_out/l1sh_$db.err
done
for c in netflix16 order4; do
timeout 900 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/l1_$c.json 2> gpurun_out/l1_$c.err; echo $c $?
python -c "
import json; d=json.load(open('gpurun_out/l1_$c.json'))
print('$c', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
done
