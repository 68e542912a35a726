export OSBLI_LIB=variants/lib_dbg.so
timeout 1500 python -m pytest tests/test_gpu_production.py tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_variants.py tests/test_gpu_symmetry.py tests/test_gpu_combinations.py -x -q -m gpu > gpurun_out/dbg_t1.log 2>&1; echo rc=$? >> gpurun_out/dbg_t1.log
OSBLI_NO_SPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_symmetry.py tests/test_gpu_combinations.py -x -q -m gpu > gpurun_out/dbg_t2.log 2>&1; echo rc=$? >> gpurun_out/dbg_t2.log
