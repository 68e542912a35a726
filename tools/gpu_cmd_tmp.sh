timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t_odd.log 2>&1; echo rc=$? >> gpurun_out/t_odd.log
OSBLI_NO_SPLIT=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_symmetry.py -x -q -m gpu > gpurun_out/t_odd_ns.log 2>&1; echo rc=$? >> gpurun_out/t_odd_ns.log
for o in 2 4 6 8 10 12; do python tools/quickbench.py 256 $o 30 2>&1 | tail -1; done > gpurun_out/orders_odd.txt
