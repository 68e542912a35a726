timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_wtma.log 2>&1; echo rc=$? >> gpurun_out/t_wtma.log
for rep in 1 2; do for o in 4 8 12; do
  python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1
  OSBLI_ZP_WTMA=0 python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1
done; done > gpurun_out/ab_wtma.txt 2>&1
