# latency-mode switch points after round 2: device time per grid search vs grid size
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
{ echo "## default"; python tools/small_threshold.py; } > gpurun_out/small_default.txt 2>&1
cp tools/libdistill_never.so paper_2110_15425_b200/libdistill.so
{ echo "## never (one thread per allocation always)"; python tools/small_threshold.py; } > gpurun_out/small_never.txt 2>&1
cat gpurun_out/small_default.txt gpurun_out/small_never.txt
