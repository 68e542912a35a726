timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_symmetry.py tests/test_gpu_slabs.py tests/test_gpu_combinations.py -x -q -m gpu > gpurun_out/t_divh.log 2>&1; echo rc=$? >> gpurun_out/t_divh.log
for rep in 1 2; do for lib in "" variants/lib_base.so; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config tgv256_o12_cons --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib cons', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['other_kernel']['avg_launch_ms'],3), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab_divh.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:divh -c 6 --csv --log-file gpurun_out/divh_launch.csv python tools/quickbench.py 256 12 2 1 c > /dev/null 2>&1
OSBLI_LIB=variants/lib_base.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:divh -c 6 --csv --log-file gpurun_out/divh_launch_base.csv python tools/quickbench.py 256 12 2 1 c > /dev/null 2>&1
