timeout 300 python bench.py --config scalar256_o12 > gpurun_out/r2f_bench_scalar.json 2> gpurun_out/r2f_bench_scalar.err
