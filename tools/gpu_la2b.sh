set -x
FT_QW_LA2=1 timeout 900 python -m pytest tests/test_quad_gpu.py -q -m gpu -x -k "quadw-chain" > gpurun_out/pytest_la2b.log 2>&1; echo pytest $?
tail -1 gpurun_out/pytest_la2b.log
for v in 1 0 1 0; do
FT_QW_LA2=$v timeout 600 python tools/time_shards.py netflix32 --P 1 2 --modes 2 > gpurun_out/la2b_$v.json 2> gpurun_out/la2b_$v.err; echo sh $v $?
grep netflix32 gpurun_out/la2b_$v.err
done
