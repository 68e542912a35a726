timeout 900 python -m pytest tests/test_gpu_symmetry.py tests/test_gpu_variants.py tests/test_gpu_combinations.py -x -q -m gpu > gpurun_out/t_symtma.log 2>&1; echo rc=$? >> gpurun_out/t_symtma.log
for c in tgv256_o12_sym tgv256_o12_sutherland tgv256_o12_cons; do for lib in "" ; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config $c --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib $c', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['other_kernel']['avg_launch_ms'],3), d['clocks']['sm_mhz'])"
OSBLI_XY_TMA=0 timeout 300 python bench.py --no-cpu-baseline --config $c --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('notma $c', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['other_kernel']['avg_launch_ms'],3), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab_symtma.txt 2>&1
