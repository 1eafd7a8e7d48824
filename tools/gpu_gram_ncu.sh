# ncu of quadw at P = 8 (mode 2 shard, producer Gram) and P = 1 (consumer Gram / per-step)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qw_p8 -f \
  python tools/time_shards.py netflix32 --P 8 --modes 2 --reps 1 > gpurun_out/qw_p8.log 2>&1; echo p8 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qw_p1 -f \
  python tools/time_shards.py netflix32 --P 1 --modes 2 --reps 1 > gpurun_out/qw_p1.log 2>&1; echo p1 $?
FT_QUADW_GRAM=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:quadw -c 1 -o gpurun_out/qw_p1_off -f \
  python tools/time_shards.py netflix32 --P 1 --modes 2 --reps 1 > gpurun_out/qw_p1_off.log 2>&1; echo p1off $?
