# tcgen05 factor sweep (K3c): parity tests, then the bench with K3c on / off
set -x
timeout 900 python -m pytest tests/test_factor_tc_gpu.py -x -q > gpurun_out/tc_tests.log 2>&1; echo tc_tests $?
tail -25 gpurun_out/tc_tests.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/tc_bench_on.json 2> gpurun_out/tc_bench_on.err; echo on $?
FT_FACTOR_TC=0 timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/tc_bench_off.json 2> gpurun_out/tc_bench_off.err; echo off $?
tail -3 gpurun_out/tc_bench_on.err
python - <<'PY'
import json
for k in ("on", "off"):
    try:
        d = json.load(open(f"gpurun_out/tc_bench_{k}.json"))
        print(k, round(d["value"]/1e9, 3), "G nnz/s", d["factor_ms"], d["core_ms"],
              {m: round(v["ms"], 3) for m, v in d["kernels"]["by_mode"].items()})
    except Exception as e:
        print(k, "failed", e)
PY
ncu --set full --clock-control none --import-source on -k regex:"factor_rows_tc" --launch-skip 4 -c 1 \
  -o gpurun_out/tc_one -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-ncu > gpurun_out/tc_one.log 2>&1
echo ncu $?
