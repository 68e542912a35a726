timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/t_tz16all.log 2>&1; echo rc=$? >> gpurun_out/t_tz16all.log
OSBLI_NO_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_symmetry.py -x -q -m gpu > gpurun_out/t_tz16ns.log 2>&1; echo rc=$? >> gpurun_out/t_tz16ns.log
for o in 2 4 6 8 10 12; do python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1; done > gpurun_out/orders_tz16.txt
timeout 300 python bench.py > gpurun_out/b_tz16.json 2>/dev/null
