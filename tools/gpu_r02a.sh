# round-2 first check: smoke, all gpu tests, bench (N=1), reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -30 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -5 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
cat gpurun_out/bench.json gpurun_out/bench_ref.json | cut -c1-3000
