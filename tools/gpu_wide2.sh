set -x
for la in 0 1; do
FT_TC_WIDE=1 FT_TCW_LA=$la timeout 600 python tools/time_shards.py netflix32 --P 1 --modes 2 > gpurun_out/w2_$la.json 2> gpurun_out/w2_$la.err; echo w $la $?
grep netflix32 gpurun_out/w2_$la.err
done
FT_TC_WIDE=1 FT_TCW_LA=0 timeout 900 python -m pytest tests/test_factor_tc_gpu.py -q -m gpu -x -k "2400 or 2300 or 3000" > gpurun_out/pytest_w2.log 2>&1; echo pytest $?
tail -2 gpurun_out/pytest_w2.log
