# ncu (source-level) of quadw's per-step form at P = 1 (bench mode 2) and P = 8 (row shard)
set -x
FT_QUADW_GRAM=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qws_p8 -f \
  python tools/time_shards.py netflix32 --P 8 --modes 2 --reps 1 > gpurun_out/qws_p8.log 2>&1; echo p8 $?
FT_QUADW_GRAM=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qws_p1 -f \
  python tools/time_shards.py netflix32 --P 1 --modes 2 --reps 1 > gpurun_out/qws_p1.log 2>&1; echo p1 $?
