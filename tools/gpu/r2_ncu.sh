# ncu captures (round 2): --set full of the three hot kernels (+ executed FP32 op counters),
# then the launch list of the default bench command.  Each command first exits 0 without ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/profile_extras.py --pp > gpurun_out/extras_plain.log 2>&1 || exit 1
NCU=/usr/local/cuda/bin/ncu
FPM=smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum
for k in pp_eval_grid_kernel ddm_batch_kernel stroop_sim_kernel; do
  $NCU --set full --metrics $FPM --import-source on --clock-control none -k regex:$k -c 1 -o gpurun_out/r02_$k -f \
      python tools/profile_extras.py --pp > gpurun_out/ncu_$k.log 2>&1
  $NCU -i gpurun_out/r02_$k.ncu-rep --page raw --csv > gpurun_out/r02_$k.raw.csv 2>/dev/null
  $NCU -i gpurun_out/r02_$k.ncu-rep --page source --csv > gpurun_out/r02_$k.source.csv 2>/dev/null
done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.json 2>&1 || exit 1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/ncu_summary.py "Round 2 — ncu --set full of the hot kernels (R10c + R22b)" gpurun_out/r02_ncu.md \
    pp=gpurun_out/r02_pp_eval_grid_kernel.raw.csv ddm=gpurun_out/r02_ddm_batch_kernel.raw.csv \
    stroop=gpurun_out/r02_stroop_sim_kernel.raw.csv > /dev/null
ls -la gpurun_out
