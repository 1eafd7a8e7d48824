# bench configs (CONFIGS) at each value (AB_VALS) of one env switch (AB_VAR)
for c in ${CONFIGS}; do for v in ${AB_VALS}; do
env ${AB_VAR}=$v timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/e_${c}_$v.json 2>gpurun_out/e_${c}_$v.err
python -c "
import json,sys; d=json.load(open('gpurun_out/e_${c}_$v.json'))
print('$c $v', round(d['value']/1e9,3), round(d['factor_ms'],2), round(d['core_ms'],2), {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items() if k.startswith('factor')})"
done; done
