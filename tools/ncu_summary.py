"""Summarise an ncu report: per kernel time, DRAM bytes, throughput, issue, occupancy."""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum', 'launch__grid_size',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = {w: (r[hdr.index(w)] if w in hdr else '') for w in WANT}
    print('%-28s t=%s ms dram R %s W %s (%s%%) issue %s%% warps %s%% regs %s inst %s fma %s alu %s lsu %s xu %s conf %s/%s' % (
        d['Kernel Name'][:28], d['gpu__time_duration.sum'], d['dram__bytes_read.sum'], d['dram__bytes_write.sum'],
        d['dram__throughput.avg.pct_of_peak_sustained_elapsed'][:5], d['smsp__issue_active.avg.pct_of_peak_sustained_active'][:5],
        d['sm__warps_active.avg.pct_of_peak_sustained_active'][:5], d['launch__registers_per_thread'],
        d['smsp__inst_executed.sum'], d['sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'][:5],
        d['sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active'][:5],
        d['sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active'][:5],
        d['sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'][:5],
        d['l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum'],
        d['l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum']))
