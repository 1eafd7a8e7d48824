# quadr with its staging space given back to L1: A/B (.so swapped) on Netflix16 and order 4
set -x
timeout 900 python -m pytest tests/test_quad_gpu.py -q -m gpu -x -k "quadr" > gpurun_out/pytest_qr.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_qr.log
cp paper_2210_06014_b200/libft_b200.so /tmp/new.so
for v in new old; do
  if [ $v = old ]; then cp _ab_old.so paper_2210_06014_b200/libft_b200.so; else cp /tmp/new.so paper_2210_06014_b200/libft_b200.so; fi
  for c in netflix16 order4; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/qr_${v}_$c.json 2> gpurun_out/qr_${v}_$c.err; echo $v $c $?
  python -c "
import json; d=json.load(open('gpurun_out/qr_${v}_$c.json'))
print('$v $c', d['value']/1e9, d['factor_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items() if 'factor' in k})"
  done
done
cp /tmp/new.so paper_2210_06014_b200/libft_b200.so
