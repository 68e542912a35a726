timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py -x -q -m gpu > gpurun_out/t_pe.log 2>&1; echo rc=$? >> gpurun_out/t_pe.log
REPS=2 STEPS=30 bash tools/ab_run.sh ab_pe.txt "4 8 10 12" cur base
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/t_pe_all.log 2>&1; echo rc=$? >> gpurun_out/t_pe_all.log
