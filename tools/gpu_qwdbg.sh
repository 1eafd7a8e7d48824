set -x
for d in 0 1 2; do
FT_QUADW_GRAM=0 FT_QW_DBG=$d timeout 600 python tools/time_shards.py netflix32 --P 1 8 --modes 2 > gpurun_out/dbg_$d.json 2> gpurun_out/dbg_$d.err; echo d $d $?
grep netflix32 gpurun_out/dbg_$d.err
done
