timeout 900 python -m pytest tests/test_gpu_tma.py -x -q -m gpu > gpurun_out/t_tma2.log 2>&1; echo rc=$? >> gpurun_out/t_tma2.log
