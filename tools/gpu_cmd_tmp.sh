timeout 900 python -m pytest tests/test_gpu_scalar.py -x -q -m gpu > gpurun_out/t_sctma.log 2>&1; echo rc=$? >> gpurun_out/t_sctma.log
for rep in 1 2; do for e in 1 0; do
OSBLI_SC_TMA=$e timeout 300 python bench.py --no-cpu-baseline --config scalar256_o12 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('tma=$e', d['value']/1e9, d['ms_per_step'], d['roofline']['frac'])"
done; done > gpurun_out/ab_sctma.txt 2>&1
