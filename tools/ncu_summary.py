import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[0]; units=rows[1]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed',
'sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum',
'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','smsp__sass_inst_executed_op_shared_ld.sum','smsp__sass_inst_executed_op_shared_st.sum',
'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__sass_thread_inst_executed_op_fadd_pred_on.sum','smsp__sass_thread_inst_executed_op_ffma_pred_on.sum','smsp__sass_thread_inst_executed_op_fmul_pred_on.sum']
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:40])
    for w in want:
        if w in hdr: print('   ',w, r[hdr.index(w)], units[hdr.index(w)])
stalls=[h for h in hdr if h.startswith('smsp__average_warp_latency_issue_stalled') or (h.startswith('smsp__warp_issue_stalled') and h.endswith('_per_warp_active.pct'))]
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:40])
    vals=sorted([(float(r[hdr.index(h)] or 0),h) for h in stalls],reverse=True)[:8]
    for v,h in vals: print('   %.2f %s'%(v,h))
print("--- stalls (warps per issue-active)")
st=[h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:40])
    vals=sorted([(float(r[hdr.index(h)] or 0),h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')) for h in st],reverse=True)[:7]
    print('   '+', '.join('%s=%.2f'%(h,v) for v,h in vals))
