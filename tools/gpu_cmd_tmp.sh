set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 300 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 300 python bench.py --no-cpu-baseline --config tgv256_o8 > gpurun_out/r2f_bench_o8.json 2>> gpurun_out/r2f_bench.err
timeout 300 python bench.py --no-cpu-baseline --config tgv64_o4 > gpurun_out/r2f_bench_o4_64.json 2>> gpurun_out/r2f_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f_bench_ref.json 2>> gpurun_out/r2f_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zpass|xypass" -s 2 -c 2 -o gpurun_out/r2f_ncu_o12 python tools/profile_step.py 256 12 1 > gpurun_out/r2f_ncu_o12.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zpass|xypass" -s 2 -c 2 -o gpurun_out/r2f_ncu_o10 python tools/profile_step.py 256 10 1 > gpurun_out/r2f_ncu_o10.log 2>&1
