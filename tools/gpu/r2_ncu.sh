# ncu captures (round 2): full sets of the three hot kernels + the bench launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:pp_eval_grid_kernel -c 1 -o gpurun_out/r02_pp -f \
    python tools/profile_extras.py --pp > gpurun_out/ncu_pp.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:ddm_batch_kernel -c 1 -o gpurun_out/r02_ddm -f \
    python tools/profile_extras.py > gpurun_out/ncu_ddm.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:stroop_sim_kernel -c 1 -o gpurun_out/r02_stroop -f \
    python tools/profile_extras.py > gpurun_out/ncu_stroop.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
for r in r02_pp r02_ddm r02_stroop; do
  $NCU -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
  $NCU -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/$r.details.csv 2>/dev/null
done
ls -la gpurun_out
