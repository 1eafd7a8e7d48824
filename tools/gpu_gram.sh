# quadw GRAM consumer: parity, bench, per-rank shard times, A/B against the per-step chain
set -x
timeout 1500 python -m pytest tests -q -m gpu -x -k "quad or netflix or parity or factor" > gpurun_out/gram_pytest.log 2>&1; echo pytest $?
tail -3 gpurun_out/gram_pytest.log
timeout 600 python bench.py --no-cpu --no-e2e --no-ncu --steps 5 > gpurun_out/gram_bench.json 2> gpurun_out/gram_bench.err; echo bench $?
FT_QUADW_GRAM=0 timeout 600 python bench.py --no-cpu --no-e2e --no-ncu --steps 5 > gpurun_out/gram_bench_off.json 2> gpurun_out/gram_bench_off.err; echo bench_off $?
timeout 900 python tools/time_shards.py netflix32 > gpurun_out/gram_shards.json 2> gpurun_out/gram_shards.err; echo shards $?
tail -4 gpurun_out/gram_shards.err
FT_QUADW_GRAM=0 timeout 900 python tools/time_shards.py netflix32 > gpurun_out/gram_shards_off.json 2> gpurun_out/gram_shards_off.err; echo shards_off $?
tail -4 gpurun_out/gram_shards_off.err
python - <<'PY'
import json
for f in ["gpurun_out/gram_bench.json", "gpurun_out/gram_bench_off.json"]:
    try:
        d = json.load(open(f))
        print(f, round(d["value"] / 1e9, 4), {k: round(v["ms"], 3) for k, v in d["kernels"]["by_mode"].items()})
    except Exception as e:
        print(f, "failed", e)
PY
