timeout 300 python bench.py > gpurun_out/bench_check.json 2> gpurun_out/bench_check.err; echo rc=$? >> gpurun_out/bench_check.err
