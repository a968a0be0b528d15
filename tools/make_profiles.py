"""Summarise ncu reports + launch lists into profiles/ (tracked).

    python tools/make_profiles.py <round-tag> <full.ncu-rep> [<more.ncu-rep> ...] --launches <csv> --bench <json>
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
     'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
     'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
     'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
     'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__block_size']


def to_bytes(v, unit):
    f = float(v.replace(',', ''))
    return f * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(unit, 1)


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith('.ncu-rep')]
    launches = sys.argv[sys.argv.index('--launches') + 1] if '--launches' in sys.argv else None
    bench = sys.argv[sys.argv.index('--bench') + 1] if '--bench' in sys.argv else None
    out_dir = os.path.join(ROOT, 'profiles')
    os.makedirs(out_dir, exist_ok=True)
    lines = ['# ncu summary (%s)' % tag, '',
             'ncu --set full --clock-control none (one launch each; cold L2, serialised).', '',
             '| kernel | time ms | DRAM read MB | DRAM write MB | DRAM % peak | issue active % | warps active % | regs | warp-inst | fma % | alu % | lsu % | grid |',
             '|---|---|---|---|---|---|---|---|---|---|---|---|---|']
    rows_json = []
    for rep in reps:
        out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {m: r[hdr.index(m)] if m in hdr else '' for m in M}
            u = {m: units[hdr.index(m)] if m in hdr else '' for m in M}
            name = r[hdr.index('Kernel Name')]
            t_ms = float(d[M[0]].replace(',', '')) * (1e-3 if u[M[0]] == 'usecond' else 1e-6 if u[M[0]] == 'nsecond' else 1)
            rd = to_bytes(d[M[1]], u[M[1]]) / 1e6
            wr = to_bytes(d[M[2]], u[M[2]]) / 1e6
            lines.append('| %s | %.4f | %.1f | %.1f | %s | %s | %s | %s | %s | %s | %s | %s | %s |' % (
                name[:48], t_ms, rd, wr, d[M[3]][:5], d[M[4]][:5], d[M[5]][:5], d[M[6]], d[M[7]],
                d[M[8]][:5], d[M[9]][:5], d[M[10]][:5], d[M[11]]))
            rows_json.append({'kernel': name, 'time_ms': t_ms, 'dram_read_MB': rd, 'dram_write_MB': wr,
                              'issue_active_pct': d[M[4]], 'inst': d[M[7]]})
    with open(os.path.join(out_dir, '%s_ncu_summary.md' % tag), 'w') as f:
        f.write('\n'.join(lines) + '\n')
    with open(os.path.join(out_dir, '%s_ncu_summary.json' % tag), 'w') as f:
        json.dump(rows_json, f, indent=1)
    if launches:
        t = defaultdict(float)
        c = defaultdict(int)
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi, mi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name'), hdr.index('Metric Unit')
        for r in rows[1:]:
            if r[mi] != 'gpu__time_duration.sum':
                continue
            scale = {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0}.get(r[ui], 1e-6)
            t[r[ki].split('(')[0]] += float(r[vi].replace(',', '')) * scale
            c[r[ki].split('(')[0]] += 1
        tot = sum(t.values())
        ll = ['# launch list (%s): `ncu --metrics gpu__time_duration.sum --clock-control none` of the bench command' % tag,
              '', 'Per-launch times are cold-cache and serialised: compare SHARES with the bench, not absolutes.', '',
              '| kernel | launches | total ms | share | avg ms |', '|---|---|---|---|---|']
        for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
            ll.append('| %s | %d | %.3f | %.1f%% | %.4f |' % (k, c[k], v, 100 * v / tot, v / c[k]))
        ll.append('| total | %d | %.3f | | |' % (sum(c.values()), tot))
        with open(os.path.join(out_dir, '%s_launches.md' % tag), 'w') as f:
            f.write('\n'.join(ll) + '\n')
        subprocess.run(['cp', launches, os.path.join(out_dir, '%s_launches.csv' % tag)])
    if bench:
        subprocess.run(['cp', bench, os.path.join(out_dir, '%s_bench.json' % tag)])


if __name__ == '__main__':
    main()
