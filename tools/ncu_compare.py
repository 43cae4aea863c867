import csv,re,sys
data=[];names=[]
for f in sys.argv[1:]:
    rows=list(csv.reader(open(f)))
    hdr=rows[0]
    for d in rows[2:]:
        data.append(dict(zip(hdr,d))); names.append(d[hdr.index('Kernel Name')][:30])
print(' '*70, ' | '.join(names))
def show(pat, minv=0):
    keys=[k for k in data[0] if re.search(pat,k)]
    for k in keys:
        try: vals=[float(d.get(k,'nan').replace(',','')) for d in data]
        except: continue
        if max(vals)>=minv: print(f"{k:80s}", ' '.join(f"{x:13.2f}" for x in vals))
show(r'sm__inst_executed_pipe_.*sum\.pct_of_peak_sustained_active$',1)
show(r'smsp__average_warps_issue_stalled_.*_per_issue_active.ratio$',0.3)
show(r'^(gpu__time_duration.sum|launch__registers_per_thread|smsp__inst_executed.sum|l1tex__data_pipe_lsu_wavefronts(_mem_shared)?.sum|l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum|l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum|l1tex__m_xbar2l1tex_read_bytes.sum|l1tex__t_sector_hit_rate.pct|sm__warps_active.avg.pct_of_peak_sustained_active|smsp__issue_active.avg.pct_of_peak_sustained_active|lts__throughput.(avg|max).pct_of_peak_sustained_elapsed|l1tex__throughput.avg.pct_of_peak_sustained_active|l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed|dram__bytes_read.sum)$')
