# ncu (source-level) of K3c-wide on Netflix mode 2 (one B200, full tensor)
set -x
FT_TC_WIDE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:factor_rows_tc -c 1 -o gpurun_out/wide_p1 -f \
  python tools/time_shards.py netflix32 --P 1 --modes 2 --reps 1 > gpurun_out/wide_p1.log 2>&1; echo p1 $?
