timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_all2.log 2>&1; echo rc=$? >> gpurun_out/t_all2.log
for o in 4 8 12; do python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1; done > gpurun_out/q_all2.txt
