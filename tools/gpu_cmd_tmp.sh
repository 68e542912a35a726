for rep in 1 2; do for lib in "" variants/lib_tmasym.so; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config tgv256_o12_sym --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib sym', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['other_kernel']['avg_launch_ms'],3), d['clocks']['sm_mhz'])"
done; done > gpurun_out/ab_sym3.txt 2>&1
