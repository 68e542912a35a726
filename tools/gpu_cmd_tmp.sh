for rep in 1 2; do for lib in "" variants/lib_ty8.so variants/lib_ty8z32.so; do
OSBLI_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --config scalar256_o12 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib', d['value']/1e9, d['ms_per_step'])"
done; done > gpurun_out/ab_sc_ty.txt 2>&1
