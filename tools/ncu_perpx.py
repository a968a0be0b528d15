"""Per-source-line lane instructions per output pixel of one kernel in an ncu report.

    python tools/ncu_perpx.py <rep> <kernel-regex> <output pixels> [min per px]
"""
import csv
import subprocess
import sys

rep, kern, px = sys.argv[1], sys.argv[2], float(sys.argv[3])
lim = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'cuda,sass', '-c', '1'], capture_output=True, text=True).stdout
cur = hdr = None
res = []
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        ie = hdr.index('Instructions Executed')
        continue
    if hdr and r and r[0] not in ('', '-') and len(r) > ie:
        try:
            res.append((cur, int(r[0]), int(r[ie] or 0), r[1][:90]))
        except ValueError:
            pass
tot = sum(x[2] for x in res)
print('lane-instr / px %.1f' % (tot * 32 / px))
for x in res:
    if x[2] * 32 / px >= lim:
        print('%-14s %5d %6.2f  %s' % (x[0], x[1], x[2] * 32 / px, x[3]))
