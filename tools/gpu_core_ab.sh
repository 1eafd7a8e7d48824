# core K4 direct-vs-staged A/B over bench configs (CONFIGS), after the quad parity tests
timeout 1500 python -m pytest tests/test_quad_gpu.py -x -q 2>&1 | tail -2
for c in ${CONFIGS:-order4 netflix16 yahoo32}; do for v in 0 1; do
FT_CORE_DIRECT=$v timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/d_${c}_$v.json 2>gpurun_out/d_${c}_$v.err
python -c "
import json,sys; d=json.load(open('gpurun_out/d_${c}_$v.json'))
print('$c $v', round(d['value']/1e9,3), round(d['factor_ms'],2), round(d['core_ms'],2), {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items() if k.startswith('core')})"
done; done
