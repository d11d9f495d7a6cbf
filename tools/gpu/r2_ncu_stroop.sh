# ncu of the trial-streaming Stroop kernel on the whole cfg4 grid (source-level: SIMT efficiency)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/profile_extras.py --stroop-full > gpurun_out/extras_full.log 2>&1 || exit 1
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:stroop_sim_kernel -s 2 -c 1 \
    -o gpurun_out/r02_stroop_full -f python tools/profile_extras.py --stroop-full > gpurun_out/ncu_sf.log 2>&1
/usr/local/cuda/bin/ncu -i gpurun_out/r02_stroop_full.ncu-rep --page source --csv > gpurun_out/r02_stroop_full.source.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i gpurun_out/r02_stroop_full.ncu-rep --page raw --csv > gpurun_out/r02_stroop_full.raw.csv 2>/dev/null
ls -la gpurun_out | grep stroop_full
