"""Per-source-line shared-memory excess wavefronts (bank conflicts) of one kernel.

    python tools/ncu_conflicts.py <rep> <kernel-regex> [top]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'cuda,sass', '-c', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
res = []
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        cur = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        cols = [i for i, h in enumerate(hdr) if 'Shared Excessive' in h or ('Shared' in h and 'Ideal' in h)]
        names = [hdr[i] for i in cols]
        continue
    if hdr and r and r[0] not in ('', '-'):
        try:
            vals = [int(float(r[i] or 0)) for i in cols]
        except (ValueError, IndexError):
            continue
        if any(vals):
            res.append((vals, cur, r[0], r[1][:80]))
print(names)
key = [i for i, n in enumerate(names) if 'Excessive' in n]
for v in sorted(res, key=lambda x: -sum(x[0][i] for i in key))[:top]:
    print(v[0], '%s:%s' % (v[1], v[2]), v[3])
