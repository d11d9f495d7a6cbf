# Memory-safety check of the kernels without compute-sanitizer (closed on this pool): the library
# built with -DDISTILL_BOUNDS_CHECK=1 (every shared-memory table / histogram index asserted in
# range; a violation traps and surfaces as a CUDA error), run over the small all-kernels driver
# and the whole GPU suite.
mkdir -p gpurun_out tools/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false \
    -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -shared -DDISTILL_BOUNDS_CHECK=1 \
    paper_2110_15425_b200/csrc/distill.cu -o tools/ab/libdistill_bounds.so
export DISTILL_LIB=$PWD/tools/ab/libdistill_bounds.so
python tools/sanitize_small.py > gpurun_out/bounds_small.log 2>&1; echo "small driver rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bounds_gputest.log 2>&1; echo "suite rc=$?"
tail -3 gpurun_out/bounds_gputest.log
