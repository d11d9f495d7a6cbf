# A/B of two library builds (tools/ab/*.so, built here with different -D flags): timing + bit-identity
mkdir -p gpurun_out
timeout 900 python tools/ab_lib.py tools/ab/lib0_base.so tools/ab/lib1_*.so --rounds 3 > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
