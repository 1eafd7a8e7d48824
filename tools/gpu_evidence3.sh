# round-2 final evidence at HEAD: gpu tests, smoke, bench, reference arm, launch list, ncu sweeps, configs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ev3_bench.json 2> gpurun_out/ev3_bench.err; echo bench $?
timeout 900 python bench.py --impl reference > gpurun_out/ev3_bench_ref.json 2> gpurun_out/ev3_bench_ref.err; echo ref $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/ev3_launches.log 2>&1
echo launches $?
ncu --set full --clock-control none --import-source on -k regex:"factor_rows|core_rows" \
  --launch-skip 12 -c 6 -o gpurun_out/ev3_sweeps -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/ev3_sweeps.log 2>&1
echo sweeps $?
ncu --set full --clock-control none --import-source on -k regex:"refresh_t" --launch-skip 6 -c 3 \
  -o gpurun_out/ev3_refresh -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-ncu > gpurun_out/ev3_refresh.log 2>&1
echo refresh $?
for c in netflix16 yahoo32 order4 order6 order10; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e --steps 3 > gpurun_out/ev3_$c.json 2> gpurun_out/ev3_$c.err; echo $c $?
done
timeout 1500 python bench.py --config order4_1b --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/ev3_order4_1b.json 2> gpurun_out/ev3_order4_1b.err; echo o41b $?
timeout 600 python bench.py --schedule hogwild --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/ev3_hogwild.json 2> gpurun_out/ev3_hogwild.err; echo hog $?
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ev3_*.json")):
    try:
        d = json.load(open(f))
        print(f, round(d["value"] / (1e9 if d.get("impl") != "reference" else 1e6), 4),
              (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"),
              {k: round(v["ms"], 2) for k, v in d.get("kernels", {}).get("by_mode", {}).items()})
    except Exception as e:
        print(f, "failed", e)
PY
