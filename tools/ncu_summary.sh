#!/bin/bash
# usage: tools/ncu_summary.sh report.ncu-rep  -> key metrics of the profiled kernel
R=$1
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
d=dict(zip(h,v))
keys=['gpu__time_duration.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active',
'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
'sm__warps_active.avg.per_cycle_active','smsp__inst_executed.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','sass__inst_executed_local_loads','sass__inst_executed_local_stores',
'dram__bytes_read.sum','dram__bytes_write.sum','lts__t_bytes.sum','launch__registers_per_thread','sm__cycles_elapsed.avg.per_second']
for k in keys: print(k, d.get(k))
st=[(k,d[k]) for k in h if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued')]
tot=sum(float(x.replace(',','') or 0) for _,x in st)
for k,x in sorted(st,key=lambda t:-float(t[1].replace(',','') or 0))[:9]: print('  %5.1f%%'%(100*float(x)/tot), k.replace('smsp__pcsamp_warps_issue_stalled_',''))
"
