# Build without Python: the library, the oracle (test infrastructure) and the C example.
# The same flags as __graft_entry__.build() / oracle.build().
NVCC ?= /usr/local/cuda/bin/nvcc
CUDA ?= /usr/local/cuda
NVCCFLAGS = -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
            -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -shared
ORACLE_CFLAGS = -O2 -std=gnu11 -ffp-contract=off -fno-fast-math -mfma -fPIC -shared -Wall

LIB = paper_2110_15425_b200/libdistill.so
ORACLE = oracle/liboracle.so

all: $(LIB) $(ORACLE) examples/c_api_demo

$(LIB): paper_2110_15425_b200/csrc/*.cu paper_2110_15425_b200/csrc/*.cuh include/distill.h
	$(NVCC) $(NVCCFLAGS) paper_2110_15425_b200/csrc/distill.cu -o $@

$(ORACLE): oracle/distill_oracle.c oracle/distill_oracle.h
	gcc $(ORACLE_CFLAGS) oracle/distill_oracle.c -o $@ -lm

examples/c_api_demo: examples/c_api_demo.c include/distill.h $(LIB)
	gcc -O2 -I include -I $(CUDA)/include $< -L paper_2110_15425_b200 -ldistill -L $(CUDA)/lib64 -lcudart \
	    -Wl,-rpath,$(CURDIR)/paper_2110_15425_b200 -o $@

clean:
	rm -f $(LIB) $(ORACLE) oracle/liboracle_count.so examples/c_api_demo

.PHONY: all clean sanitize-oracle

# ASan + UBSan run of the CPU oracle: instrumented copies of
# liboracle*.so, the oracle's CPU test suite under the preloaded runtime.
sanitize-oracle:
	DISTILL_ORACLE_SANITIZE=1 LD_PRELOAD="$$(gcc -print-file-name=libasan.so) $$(gcc -print-file-name=libubsan.so)" \
	ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 \
	python -m pytest tests/test_oracle_rng.py tests/test_oracle_pp.py tests/test_oracle_argmax.py \
	    tests/test_oracle_ddm_lca.py tests/test_oracle_episode.py tests/test_oracle_amr.py \
	    tests/test_oracle_ext_stroop.py tests/test_oracle_exact_law.py -q -p no:cacheprovider
