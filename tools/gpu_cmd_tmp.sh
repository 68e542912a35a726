for rep in 1 2; do for o in 8 12; do
python tools/quickbench.py 256 $o 30 2 2>&1 | tail -n 1
OSBLI_LIB=variants/lib_mixbtr.so python tools/quickbench.py 256 $o 30 2 2>&1 | tail -n 1
done; done > gpurun_out/ab_mixbtr.txt 2>&1
