"""Summarise an ncu report: key metrics per kernel + stall share per code region.
Usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'launch__registers_per_thread', 'sm__warps_active.avg.per_cycle_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'smsp__inst_executed.sum', 'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum']
for r in rows[2:]:
    print('----', r[h.index('Kernel Name')][:60])
    for k in keys:
        if k in h:
            print(f"  {k} = {r[h.index(k)]} {rows[1][h.index(k)]}")
    st = [(x, float(r[i] or 0)) for i, x in enumerate(h) if 'average_warps_issue_stalled' in x]
    st = sorted([s for s in st if s[1] > 0.15], key=lambda s: -s[1])
    print('  stalls/issue:', ', '.join(f"{s[0].split('stalled_')[1].split('_per')[0]}={s[1]:.2f}" for s in st))
