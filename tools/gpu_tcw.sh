set -x
timeout 1200 python -m pytest tests/test_factor_tc_gpu.py tests/test_netflix_parity_gpu.py -q -x > gpurun_out/tcw_tests.log 2>&1; echo tests $?
tail -15 gpurun_out/tcw_tests.log
timeout 600 python bench.py --no-cpu --no-e2e --no-ncu > gpurun_out/tcw_bench.json 2> gpurun_out/tcw_bench.err; echo bench $?
tail -3 gpurun_out/tcw_bench.err
python -c "
import json; d=json.load(open('gpurun_out/tcw_bench.json'))
print(d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
