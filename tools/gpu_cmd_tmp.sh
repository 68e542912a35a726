REPS=2 STEPS=30 bash tools/ab_run.sh ab_st8.txt "4 8 10 12" cur st8
for rep in 1 2; do for lib in "" variants/lib_st8.so; do for c in tgv256_o12_sym; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config $c --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('$lib $c', round(d['value']/1e9,3), round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['other_kernel']['avg_launch_ms'],3), d['clocks']['sm_mhz'])"
done; done; done >> gpurun_out/ab_st8.txt 2>&1
