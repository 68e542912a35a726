timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/t_final2.log 2>&1; echo rc=$? >> gpurun_out/t_final2.log
