# round evidence: bench line, reference arm, launch list, ncu --set full of the sweeps + refresh
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench $?
timeout 900 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo ref $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/ev_launches.log 2>&1
echo launches $?
ncu --set full --clock-control none --import-source on -k regex:"factor_rows|core_rows" \
  --launch-skip 12 -c 6 -o gpurun_out/ev_sweeps -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/ev_sweeps.log 2>&1
echo sweeps $?
ncu --set full --clock-control none --import-source on -k regex:"refresh_tc" --launch-skip 6 -c 3 \
  -o gpurun_out/ev_refresh -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/ev_refresh.log 2>&1
echo refresh $?
python -c "
import json
for f in ('gpurun_out/ev_bench.json', 'gpurun_out/ev_bench_ref.json'):
    try:
        d = json.load(open(f)); print(f, d['value']/1e9 if d.get('impl') != 'reference' else d['value'], d.get('e2e', {}).get('value'), d.get('roofline', {}) and d['roofline'].get('frac'))
    except Exception as e: print(f, 'failed', e)
"
