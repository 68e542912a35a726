timeout 1500 python -m pytest tests/test_gpu_production.py -x -q -m gpu > gpurun_out/t_prod.log 2>&1; echo rc=$? >> gpurun_out/t_prod.log
