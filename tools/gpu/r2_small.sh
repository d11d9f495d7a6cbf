# latency-mode switch points after round 2: device time per grid search vs grid size
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true \
    -prec-sqrt=true -Xcompiler -fPIC -shared -DDISTILL_PP_SMALL_MODE=0 paper_2110_15425_b200/csrc/distill.cu \
    -o tools/libdistill_never.so
{ echo "## default"; python tools/small_threshold.py; } > gpurun_out/small_default.txt 2>&1
cp tools/libdistill_never.so paper_2110_15425_b200/libdistill.so
{ echo "## never (one thread per allocation always)"; python tools/small_threshold.py; } > gpurun_out/small_never.txt 2>&1
cat gpurun_out/small_default.txt gpurun_out/small_never.txt
