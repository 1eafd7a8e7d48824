# A/B of one env switch: quad parity tests, then a short bench with the switch at each value
# usage: AB_VAR=FT_QUADR_DEDUP AB_VALS="0 1" bash tools/gpu_ab.sh
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py -x -q > gpurun_out/ab_tests.log 2>&1; echo quad_tests $?
tail -3 gpurun_out/ab_tests.log
for v in ${AB_VALS}; do
env ${AB_VAR}=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; echo bench $v $?
python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
done
