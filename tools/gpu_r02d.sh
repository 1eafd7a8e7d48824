set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "hogwild" > gpurun_out/d_hog.log 2>&1; echo hog $?
tail -3 gpurun_out/d_hog.log
python tools/time_e2e_parts.py > gpurun_out/d_e2e_parts.log 2>&1; tail -8 gpurun_out/d_e2e_parts.log
timeout 1500 python bench.py --config order4_1b --no-cpu --no-e2e --no-ncu --steps 3 > gpurun_out/d_order4_1b.json 2> gpurun_out/d_order4_1b.err; echo o41b $?
tail -4 gpurun_out/d_order4_1b.err
python -c "
import json; d=json.load(open('gpurun_out/d_order4_1b.json'))
print(d['value']/1e9, d['factor_ms'], d['core_ms'], {k: round(v['ms'],3) for k,v in d['kernels']['by_mode'].items()})"
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
