timeout 1500 python -m pytest tests/test_quad_gpu.py -x -q 2>&1 | tail -3
rm -f gpurun_out/b_*.json
for c in ${CONFIGS:-netflix32 order4 order6}; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; echo $c $?
done
for f in gpurun_out/b_*.json; do python -c "
import json,sys; d=json.load(open('$f'))
print('$f', round(d['value']/1e9,3), round(d['factor_ms'],2), round(d['core_ms'],2), {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"; done
