# quick GPU iteration: new-kernel parity tests + a short bench per factor variant (outputs in gpurun_out/)
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py -x -q > gpurun_out/quad_tests.log 2>&1; echo quad_tests $?
tail -15 gpurun_out/quad_tests.log
for v in auto quadw; do
FT_FACTOR_KERNEL=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo bench $v $?
python -c "
import json; d=json.load(open('gpurun_out/bench_$v.json'))
print('$v', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
done
