# the N>1 bench path on one GPU: two ranks share cuda:0 over gloo (timings meaningless)
set -x
FT_DIST_BACKEND=gloo FT_PEER=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/dist2.json 2> gpurun_out/dist2.err
echo dist $?
tail -3 gpurun_out/dist2.err; cat gpurun_out/dist2.json
