timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/t_final.log 2>&1; echo rc=$? >> gpurun_out/t_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; echo rc=$? >> gpurun_out/smoke_final.log
