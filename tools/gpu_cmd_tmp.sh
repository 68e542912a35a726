timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_production.py tests/test_gpu_tma.py -x -q -m gpu > gpurun_out/t_qsp.log 2>&1; echo rc=$? >> gpurun_out/t_qsp.log
REPS=3 STEPS=30 bash tools/ab_run.sh ab_qsp2.txt "4 8 12" cur noqsp
