# L2-only gathers of the large C matrices (K4 direct: ld.global.nc.L1::no_allocate; K3c: cp.async.cg)
set -x
for na in 1 0; do
FT_L1_STREAM=$na timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/l1b_$na.json 2> gpurun_out/l1b_$na.err; echo bench na=$na $?
python -c "
import json; d=json.load(open('gpurun_out/l1b_$na.json'))
print('na=$na', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()}, d['train_rmse'])"
done
timeout 900 python -m pytest tests/test_factor_tc_gpu.py tests/test_netflix_parity_gpu.py -q -m gpu -x > gpurun_out/pytest_l1b.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_l1b.log
