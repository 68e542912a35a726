timeout 600 python tools/tgv_history.py gpurun_out/r2z_tgv64_o4_history.csv > gpurun_out/hist.log 2>&1; echo rc=$? >> gpurun_out/hist.log
