"""Summarise ncu reports, the bench launch list and bench lines into profiles/.

    python tools/make_profiles.py <tag> --full <rep>:<op,op,...> [--full ...]
                                  --launches <csv> --bench <json> [<json> ...]

Each --full report must hold the main kernels of the listed cfg2 transforms in
launch order (tools/profile_ops.py --ops <same list> --reps 1, captured with a
kernel regex that skips k_prep / k_affine_setup / k_eq_lut).  Writes
  profiles/<tag>_ncu_summary.md     per-kernel table (time, DRAM traffic, issue, ...)
  profiles/ncu_traffic.json         cfg2 op -> measured DRAM bytes per launch (read by bench.py)
  profiles/<tag>_launches.md/.csv   launch list of the bench command (kernel shares)
  profiles/<tag>_bench_*.json       the bench lines
"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
     'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
     'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'smsp__inst_executed.sum',
     'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
     'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
     'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'launch__grid_size', 'launch__block_size']
SCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0,
         'ns': 1e-6, 'us': 1e-3, 'ms': 1.0}
KERNELS_PER_OP = {}  # kernels per transform in the capture order (Equalize is one fused kernel since r2)
PEAK = json.load(open(os.path.join(ROOT, 'MEASURED_PEAKS.json')))['hbm_gbs'] if os.path.exists(
    os.path.join(ROOT, 'MEASURED_PEAKS.json')) else 6650.0


def num(v, unit):
    return float(v.replace(',', '')) * SCALE.get(unit, 1.0)


def read_rep(rep):
    """kernels of an ncu report (.ncu-rep) or of its raw-page CSV (made on the box)"""
    if rep.endswith('.csv'):
        out = open(rep).read()
    else:
        out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for m in M:
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[m] = num(r[i], units[i])
                except ValueError:
                    d[m] = r[i]
        d['name'] = r[hdr.index('Kernel Name')]
        res.append(d)
    return res


def main():
    args = sys.argv[1:]
    tag = args[0]
    fulls, launches, benches, comps = [], None, [], []
    i = 1
    while i < len(args):
        if args[i] == '--full':
            rep, _, ops = args[i + 1].partition(':')
            fulls.append((rep, ops.split(',')))
            i += 2
        elif args[i] == '--comp':  # a report of other kernels: one table row per kernel
            comps.append(args[i + 1])
            i += 2
        elif args[i] == '--launches':
            launches = args[i + 1]
            i += 2
        elif args[i] == '--bench':
            i += 1
            while i < len(args) and not args[i].startswith('--'):
                benches.append(args[i])
                i += 1
        else:
            raise SystemExit('bad arg ' + args[i])
    out_dir = os.path.join(ROOT, 'profiles')
    os.makedirs(out_dir, exist_ok=True)
    lines = ['# ncu summary (%s): cfg2 corpus (2000 ragged RGB images, 913 MB), one launch per kernel' % tag, '',
             '`ncu --set full --clock-control none` of `tools/profile_ops.py --ops <op> --reps 1` on one B200; '
             'cold L2, serialised (compare with bench shares, not absolutes).  DRAM columns are measured '
             'traffic; algorithmic bytes for the same-shape ops are 915 MB read + 863 MB write.', '',
             '| transform | kernel | time ms | DRAM read MB | DRAM write MB | DRAM GB/s | issue active % | '
             'warps active % | regs | warp-inst | inst / out px | FMA pipe % | ALU pipe % |',
             '|---|---|---|---|---|---|---|---|---|---|---|---|---|']
    traffic = {}
    px = {'RandomCrop64': 2000 * 64 * 64, 'PadToSize512': 2000 * 512 * 512, 'Resize512': 2000 * 512 * 512,
          'RandomSizedCrop64-512': 2000 * 512 * 512}
    sys.path.insert(0, ROOT)
    from synth import gen
    same = sum(h * w for h, w in gen.cfg2_sizes(2000))  # cfg2 corpus pixels
    for rep, ops in fulls:
        ks = read_rep(rep)
        k = 0
        for op in ops:
            n = KERNELS_PER_OP.get(op, 1)
            grp = ks[k:k + n]
            k += n
            tot_r = tot_w = 0.0
            for d in grp:
                t = d.get(M[0], 0.0)
                rd = d.get(M[1], 0.0) / 1e6
                wr = d.get(M[2], 0.0) / 1e6
                tot_r += rd
                tot_w += wr
                inst = d.get(M[7], 0.0)
                lines.append('| %s | %s | %.4f | %.1f | %.1f | %.0f | %.1f | %.1f | %d | %.3g | %.2f | %.1f | %.1f |' % (
                    op, d['name'].split('(')[0][:40], t, rd, wr, (rd + wr) / t if t else 0.0, d.get(M[4], 0.0), d.get(M[5], 0.0),
                    int(d.get(M[6], 0)), inst, inst * 32.0 / px.get(op, same), d.get(M[8], 0.0), d.get(M[9], 0.0)))
            traffic[op] = round((tot_r + tot_w) * 1e6)
    if fulls:
        with open(os.path.join(out_dir, '%s_ncu_summary.md' % tag), 'w') as f:
            f.write('\n'.join(lines) + '\n\n"inst / out px" = lane instructions (warp instructions x 32) per output '
                    'pixel.\n')
        tj = os.path.join(out_dir, 'ncu_traffic.json')
        old = json.load(open(tj)) if os.path.exists(tj) else {}
        old['cfg2'] = traffic
        old['note'] = ('dram__bytes_read.sum + dram__bytes_write.sum per launch of each transform\'s kernels '
                       '(ncu --set full, %s)' % tag)
        with open(tj, 'w') as f:
            json.dump(old, f, indent=1)
    if comps:
        cl = ['# ncu summary (%s): kernels of the composed configs and the next-row transforms' % tag, '',
              '`ncu --set full --clock-control none`, one launch per kernel, cold L2 (see tools/gpu_r2_ncu.sh '
              'for the commands: cfg3 Rotate with masks, cfg4 fused Compose, cfg5 co-transform with masks and '
              'boxes; Rot90, GridDistortion, ElasticTransform on 500 cfg2 images).', '',
              '| report | kernel | time ms | DRAM read MB | DRAM write MB | DRAM GB/s | frac of %.0f GB/s | '
              'issue active %% | warps active %% | regs | warp-inst | FMA pipe %% | ALU pipe %% |' % PEAK,
              '|---|---|---|---|---|---|---|---|---|---|---|---|---|']
        for rep in comps:
            for d in read_rep(rep):
                t = d.get(M[0], 0.0)
                rd = d.get(M[1], 0.0) / 1e6
                wr = d.get(M[2], 0.0) / 1e6
                gbs = (rd + wr) / t if t else 0.0
                cl.append('| %s | %s | %.4f | %.1f | %.1f | %.0f | %.3f | %.1f | %.1f | %d | %.3g | %.1f | %.1f |' % (
                    os.path.basename(rep).replace('_raw.csv', ''), d['name'].split('(')[0][:48], t, rd, wr, gbs,
                    gbs / PEAK, d.get(M[4], 0.0), d.get(M[5], 0.0), int(d.get(M[6], 0)), d.get(M[7], 0.0),
                    d.get(M[8], 0.0), d.get(M[9], 0.0)))
        with open(os.path.join(out_dir, '%s_ncu_comp.md' % tag), 'w') as f:
            f.write('\n'.join(cl) + '\n')
    if launches:
        t = defaultdict(float)
        c = defaultdict(int)
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        hdr = rows[0]
        ki, vi, mi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name'), hdr.index('Metric Unit')
        for r in rows[1:]:
            if r[mi] != 'gpu__time_duration.sum':
                continue
            key = r[ki].split('(')[0]
            t[key] += num(r[vi], r[ui])
            c[key] += 1
        tot = sum(t.values())
        ll = ['# launch list (%s): `ncu --metrics gpu__time_duration.sum --clock-control none` of '
              '`python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 0`' % tag, '',
              'Per-launch times are cold-cache and serialised: compare SHARES with the bench, not absolutes.', '',
              '| kernel | launches | total ms | share | avg ms |', '|---|---|---|---|---|']
        for kname, v in sorted(t.items(), key=lambda kv: -kv[1]):
            ll.append('| %s | %d | %.3f | %.1f%% | %.4f |' % (kname, c[kname], v, 100 * v / tot, v / c[kname]))
        ll.append('| total | %d | %.3f | | |' % (sum(c.values()), tot))
        with open(os.path.join(out_dir, '%s_launches.md' % tag), 'w') as f:
            f.write('\n'.join(ll) + '\n')
        shutil.copy(launches, os.path.join(out_dir, '%s_launches.csv' % tag))
    for b in benches:
        shutil.copy(b, os.path.join(out_dir, '%s_%s' % (tag, os.path.basename(b))))


if __name__ == '__main__':
    main()
