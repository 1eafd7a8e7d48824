# K4 direct A/B: the working-tree .so vs _ab_old.so (swapped in place), plus the K4 parity tests
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_k4acc.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_k4acc.log
cp paper_2210_06014_b200/libft_b200.so /tmp/new.so
for v in new old new old; do
  if [ $v = old ]; then cp _ab_old.so paper_2210_06014_b200/libft_b200.so; else cp /tmp/new.so paper_2210_06014_b200/libft_b200.so; fi
  timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/k4_$v.json 2> gpurun_out/k4_$v.err; echo bench $v $?
  python -c "
import json; d=json.load(open('gpurun_out/k4_$v.json'))
print('$v', d['value']/1e9, d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items() if 'core' in k})"
done
cp /tmp/new.so paper_2210_06014_b200/libft_b200.so
for c in netflix16; do
timeout 900 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/k4_$c.json 2> gpurun_out/k4_$c.err; echo $c $?
python -c "
import json; d=json.load(open('gpurun_out/k4_$c.json'))
print('$c', d['value']/1e9, d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items() if 'core' in k})"
done
