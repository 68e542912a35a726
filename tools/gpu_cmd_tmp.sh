for c in tgv256_o12_sym tgv256_o12_sutherland tgv256_o12_rk3_2r; do timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/r2z_bench_$c.json 2>> gpurun_out/r2z.err; done
