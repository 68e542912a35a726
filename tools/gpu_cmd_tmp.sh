timeout 900 ncu --set full --clock-control none -k regex:"xypass" -s 2 -c 1 -o gpurun_out/sym_cur python tools/profile_sym.py > gpurun_out/sym_cur.log 2>&1
OSBLI_LIB=variants/lib_tmasym.so timeout 900 ncu --set full --clock-control none -k regex:"xypass" -s 2 -c 1 -o gpurun_out/sym_tma python tools/profile_sym.py > gpurun_out/sym_tma.log 2>&1
