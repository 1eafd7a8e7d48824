# scaling-model inputs with HEAD's kernels: per-rank shard sweeps, Netflix32, P = 1, 2, 4, 8
set -x
timeout 900 python tools/time_shards.py netflix32 --P 1 2 4 8 > gpurun_out/shards_final.json 2> gpurun_out/shards_final.err; echo sh $?
grep netflix32 gpurun_out/shards_final.err
