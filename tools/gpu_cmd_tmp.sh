timeout 1200 python tools/oracle_fullsize.py gpurun_out/r2z_oracle_fullsize_256_o12.json 256 12 > gpurun_out/ofs.log 2>&1; echo rc=$? >> gpurun_out/ofs.log
