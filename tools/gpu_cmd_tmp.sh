timeout 300 python bench.py > gpurun_out/r2t_bench_tgv256_o12.json 2> gpurun_out/r2t.err
timeout 300 python bench.py --no-cpu-baseline --config tgv256_o8 > gpurun_out/r2t_bench_tgv256_o8.json 2>> gpurun_out/r2t.err
for c in tgv256_o12_sym tgv256_o12_sutherland tgv256_o12_cons tgv256_o12_rk3_2r tgv256_o12_slab1 tgv64_o4; do timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/r2t_bench_$c.json 2>> gpurun_out/r2t.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2t_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zpass" -s 2 -c 1 -o gpurun_out/r2t_ncu_z python tools/profile_step.py 256 12 1 > gpurun_out/r2t_ncu_z.log 2>&1
