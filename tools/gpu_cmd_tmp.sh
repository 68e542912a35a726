timeout 1200 python -m pytest tests/test_gpu_slabs.py -x -q -m gpu > gpurun_out/t_slabs.log 2>&1; echo rc=$? >> gpurun_out/t_slabs.log
