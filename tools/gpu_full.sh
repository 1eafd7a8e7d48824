# full GPU check: all gpu tests, smoke, bench (outputs in gpurun_out/)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench $?
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json'))
print(d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
