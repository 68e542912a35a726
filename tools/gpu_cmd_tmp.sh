nvidia-smi --query-gpu=name,serial,clocks.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi2.txt
for r in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/rep_$r.json 2>/dev/null; done
for o in 12; do python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1; done > gpurun_out/rep_q.txt
