"""Key raw metrics of every kernel in an ncu report (time, DRAM, issue, stalls)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ''
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'sm__cycles_elapsed.avg', 'smsp__cycles_active.avg']
stalls = [c for c in h if c.startswith('smsp__average_warps_issue_stalled_') and c.endswith('_per_issue_active.ratio')]
for r in rows[2:]:
    name = r[h.index('Kernel Name')]
    if flt and flt not in name:
        continue
    print('==', name[:90])
    for w in want:
        if w in h:
            print('   %-70s %s' % (w, r[h.index(w)]))
    st = sorted(((float(r[h.index(c)] or 0), c) for c in stalls), reverse=True)[:8]
    print('   stalls:', ', '.join('%s %.2f' % (c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), v) for v, c in st))
