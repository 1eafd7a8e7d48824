# quadw lookahead A/B + full GPU suite
set -x
for la in 1 0; do
FT_QUADW_LA=$la timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/la_$la.json 2> gpurun_out/la_$la.err; echo bench la=$la $?
python -c "
import json; d=json.load(open('gpurun_out/la_$la.json'))
print('la=$la', d['value']/1e9, d['factor_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -5 gpurun_out/pytest_gpu.log
