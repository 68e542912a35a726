timeout 300 python bench.py > gpurun_out/r2z_bench_tgv256_o12.json 2> gpurun_out/r2z.err
timeout 300 python bench.py --no-cpu-baseline --config tgv256_o8 > gpurun_out/r2z_bench_tgv256_o8.json 2>> gpurun_out/r2z.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2z_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_ncu_launch.log 2>&1
for o in 2 4 6 8 10 12; do python tools/quickbench.py 256 $o 30 2>&1 | tail -n 1; done > gpurun_out/r2z_orders.txt
