timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_xtma_all.log 2>&1; echo rc=$? >> gpurun_out/t_xtma_all.log
OSBLI_NO_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_combinations.py -x -q -m gpu > gpurun_out/t_xtma_ns.log 2>&1; echo rc=$? >> gpurun_out/t_xtma_ns.log
timeout 300 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
timeout 300 python bench.py --no-cpu-baseline --config tgv256_o8 > gpurun_out/r2g_bench_o8.json 2>> gpurun_out/r2g_bench.err
