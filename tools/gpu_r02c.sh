set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo bench $?
python tools/time_e2e_parts.py > gpurun_out/c_e2e_parts.log 2>&1; tail -15 gpurun_out/c_e2e_parts.log
python -c "
import json; d=json.load(open('gpurun_out/c_bench.json'))
print(d['value']/1e9, d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['roofline']['frac'], d['cpu_baseline']['value'])"
