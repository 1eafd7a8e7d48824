# full GPU check: all gpu tests, smoke, bench (outputs in gpurun_out/)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -15 gpurun_out/pytest_gpu.log
python tools/time_e2e_parts.py > gpurun_out/e2e_parts.log 2>&1; cat gpurun_out/e2e_parts.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value']/1e9, d['factor_ms'], d['core_ms'], d['e2e']['value']/1e9, {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
