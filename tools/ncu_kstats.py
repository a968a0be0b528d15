"""Kernel-level stats of the first matching kernel in an ncu report: time, DRAM, issue,
occupancy, instructions per output pixel, and the warp-stall breakdown.
    python tools/ncu_kstats.py <rep> <kernel-regex> [out_px]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
px = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv', '--kernel-name', 'regex:' + kern, '-c', '1'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}


def g(k):
    x = d.get(k, ('nan', ''))[0].replace(',', '')
    try:
        return float(x)
    except ValueError:
        return float('nan')


print(d.get('Kernel Name', ('?',))[0][:80])
for k in ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
          'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
          'launch__occupancy_limit_warps', 'launch__shared_mem_per_block_dynamic', 'smsp__inst_executed.sum',
          'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
          'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
          'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']:
    print('  %-60s %s %s' % (k, d.get(k, ('-', ''))[0], d.get(k, ('', ''))[1]))
if px:
    print('  lane-instr / out px: %.2f' % (g('smsp__inst_executed.sum') * 32 / px))
st = [(g(k), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''))
      for k in d if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
print('  stalls per issue:', ', '.join('%s %.2f' % (n, x) for x, n in sorted(st, reverse=True)[:8]))
