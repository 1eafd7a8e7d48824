set -x
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_factor_tc_gpu.py -q -x > gpurun_out/dist_tests.log 2>&1; echo dist $?
tail -5 gpurun_out/dist_tests.log
timeout 1200 python tools/hogwild_ab.py > gpurun_out/hogwild_ab.log 2>&1; echo hog $?
tail -8 gpurun_out/hogwild_ab.log
timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/bench_q.json 2>/dev/null; echo bench $?
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print(d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
