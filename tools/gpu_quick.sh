# quick GPU iteration: a short bench per factor variant (outputs in gpurun_out/)
set -x
for v in ${VARIANTS:-auto}; do
FT_FACTOR_KERNEL=$v timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo bench $v $?
python -c "
import json; d=json.load(open('gpurun_out/bench_$v.json'))
print('$v', d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
done
