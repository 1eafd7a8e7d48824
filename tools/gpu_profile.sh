# round evidence: bench line, reference arm, launch list, ncu --set full of the sweeps and aux
# kernels, secondary configs (run under gpurun; outputs in gpurun_out/)
set -x
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
echo launches $?
ncu --set full --clock-control none --import-source on -k regex:"factor_rows|core_rows" \
  --launch-skip 18 -c 6 -o gpurun_out/sweeps -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/sweeps_bench.log 2>&1
echo sweeps $?
ncu --set full --clock-control none -k regex:"refresh_tc|decode_levels|pack_keys_vals|pack_derived|decode_derived|leaf_pc_kernel" \
  -c 10 -o gpurun_out/aux -f python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/aux_bench.log 2>&1
echo aux $?
for c in netflix16 yahoo32 order6 order4; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; echo $c $?
done
