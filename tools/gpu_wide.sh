# K3c-wide (quad-layout consumers) parity + Netflix mode-2 A/B
set -x
timeout 900 python -m pytest tests/test_factor_tc_gpu.py -q -m gpu -x > gpurun_out/pytest_wide.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_wide.log
for w in 1 0; do
FT_TC_WIDE=$w timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/wide_$w.json 2> gpurun_out/wide_$w.err; echo bench wide=$w $?
python -c "
import json; d=json.load(open('gpurun_out/wide_$w.json'))
print('wide=$w', d['value']/1e9, d['factor_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()}, d['train_rmse'], d['test_rmse'])"
done
