set -x
timeout 1200 python -m pytest tests -q -m gpu -x -k "build or layout or tree or golden or derived or config1 or order or drop or fibers or netflix" > gpurun_out/b_pytest.log 2>&1; echo pytest $?
tail -2 gpurun_out/b_pytest.log
timeout 600 python tools/prof_build.py 2>&1 | tail -22
timeout 900 python bench.py --no-cpu --no-ncu --steps 5 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo bench $?
python -c "import json; d=json.load(open('gpurun_out/b_bench.json')); print(d['value']/1e9, d['e2e'])"
