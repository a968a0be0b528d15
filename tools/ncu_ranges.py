"""Sum an ncu source page (instructions executed, stall samples) over line ranges.

    python tools/ncu_ranges.py <rep> <kernel-regex> file:a-b[=label] ...
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'cuda,sass', '-c', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
per = {}
cur = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        ie = hdr.index('Instructions Executed')
        ws = hdr.index('Warp Stall Sampling (All Samples)')
        continue
    if hdr and r and r[0] not in ('', '-') and len(r) > ie:
        try:
            per[(cur, int(r[0]))] = (int(r[ie] or 0), int(r[ws] or 0))
        except ValueError:
            pass
tot = sum(v[0] for v in per.values())
tots = sum(v[1] for v in per.values())
print('total warp-inst %d  stall samples %d' % (tot, tots))
seen = set()
for spec in sys.argv[3:]:
    rng, _, label = spec.partition('=')
    f, _, ab = rng.partition(':')
    a, _, b = ab.partition('-')
    a, b = int(a), int(b or a)
    keys = [k for k in per if k[0] == f and a <= k[1] <= b]
    seen.update(keys)
    s = sum(per[k][0] for k in keys)
    t = sum(per[k][1] for k in keys)
    print('%-28s %5.1f%% inst  %5.1f%% stall' % (label or spec, 100.0 * s / tot, 100.0 * t / max(tots, 1)))
rest = [k for k in per if k not in seen]
print('%-28s %5.1f%% inst  %5.1f%% stall' % ('(other)', 100.0 * sum(per[k][0] for k in rest) / tot,
                                              100.0 * sum(per[k][1] for k in rest) / max(tots, 1)))
for k in sorted(rest, key=lambda k: -per[k][0])[:15]:
    print('   %s:%d %.1f%%' % (k[0], k[1], 100.0 * per[k][0] / tot))
