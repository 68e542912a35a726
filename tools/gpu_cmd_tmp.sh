for rep in 1 2; do for lib in "" variants/lib_za1.so variants/lib_za0.so variants/lib_scv2.so; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config scalar256_o12 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done; done > gpurun_out/sc_ab2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_scalar.py -x -q -m gpu > gpurun_out/t_sc.log 2>&1; echo rc=$? >> gpurun_out/t_sc.log
