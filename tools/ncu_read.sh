#!/bin/bash
# summarise a report from tools/ncu_one.sh: hot source lines + stall reasons (dev tool)
rep=$1
ncu -i $rep --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_mix.csv
python "$(dirname "$0")/src_hot.py" /tmp/_mix.csv ${2:-25}
ncu -i $rep --page raw --csv 2>/dev/null > /tmp/_raw.csv
python - <<'PY'
import csv
rows=list(csv.reader(open('/tmp/_raw.csv')))
h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
d=dict(zip(h,v))
st={k.replace('smsp__pcsamp_warps_issue_stalled_',''):float(d[k]) for k in h if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued') and d[k] not in ('','0')}
tot=sum(st.values()) or 1
print('stalls:', ', '.join(f"{k} {100*x/tot:.0f}%" for k,x in sorted(st.items(), key=lambda a:-a[1]) if x/tot>0.01))
for k in ['gpu__time_duration.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:
    print(k, d.get(k))
PY
