timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_diag.log 2>&1; echo rc=$? >> gpurun_out/t_diag.log
for c in tgv256_o12 tgv256_o8; do timeout 300 python bench.py --no-cpu-baseline --config $c --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c', d['value']/1e9, d['diagnostics'])"; done > gpurun_out/diag_bench.txt 2>&1
