for v in auto quadw quadrp; do
  if [ $v = auto ]; then E=""; else E="FT_FACTOR_KERNEL=$v"; fi
  env $E timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err; echo bench $v $?
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', d['value']/1e9, d['factor_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()}, d['train_rmse'])" 2>&1 | tail -1
done
