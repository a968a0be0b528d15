"""Top SASS instructions by stall samples with their dominant stall reasons, plus the
instructions just before them.   python tools/ncu_stalls.py <rep> <kernel-regex> [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'sass', '-c', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]
ws = h.index('Warp Stall Sampling (All Samples)')
src = h.index('Source')
sc = [(i, c) for i, c in enumerate(h) if c.startswith('stall_') and '(' not in c]
body = [r for r in rows[hi + 1:] if len(r) > ws]
tot = sum(int(r[ws] or 0) for r in body)
order = sorted(range(len(body)), key=lambda k: -int(body[k][ws] or 0))[:top]
for k in order:
    r = body[k]
    reasons = sorted(((int(r[i] or 0), c[6:]) for i, c in sc), reverse=True)[:3]
    print('%5.1f%%  %-60s %s' % (100.0 * int(r[ws] or 0) / tot, r[src][:60],
                                 ' '.join('%s:%d' % (c, v) for v, c in reasons if v)))
    for rr in body[max(0, k - 3):k]:
        print('            prev: %s' % rr[src][:70])
