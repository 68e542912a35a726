mkdir -p gpurun_out
for rep in 1 2; do for lib in "" variants/lib_base.so; do for a in "1 v" "2" "1"; do OSBLI_LIB=$lib python tools/quickbench.py 256 12 40 $a 2>&1 | tail -1; done; done; done > gpurun_out/ab7.txt
