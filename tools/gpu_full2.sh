# full GPU check: smoke, all gpu tests (outputs in gpurun_out/)
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -25 gpurun_out/pytest_gpu.log
