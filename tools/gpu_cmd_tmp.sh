timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -x -q -m gpu > gpurun_out/t_tma.log 2>&1; echo rc=$? >> gpurun_out/t_tma.log
for rep in 1 2; do for o in 4 8 12; do
  python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1
  OSBLI_ZP_TMA=0 python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1
done; done > gpurun_out/ab_tma2.txt 2>&1
