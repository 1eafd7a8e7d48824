# K3c on / off on the other BASELINE shapes (per-mode kernel ms), then order10 / order4_1b
set -x
for c in netflix16 yahoo32 order4 order6; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/ab_${c}_on.json 2> gpurun_out/ab_${c}_on.err; echo $c on $?
  FT_FACTOR_TC=0 timeout 900 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/ab_${c}_off.json 2> gpurun_out/ab_${c}_off.err; echo $c off $?
done
for c in order10 order4_1b; do
  timeout 1200 python bench.py --config $c --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/ab_${c}_on.json 2> gpurun_out/ab_${c}_on.err; echo $c $?
  tail -3 gpurun_out/ab_${c}_on.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    try:
        d = json.load(open(f))
        print(f.split("/")[-1], round(d["value"]/1e9, 3), "G nnz/s", round(d["factor_ms"],2), round(d["core_ms"],2),
              {m: round(v["ms"], 2) for m, v in d["kernels"]["by_mode"].items()})
    except Exception as e:
        print(f, "failed", e)
PY
