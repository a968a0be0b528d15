"""Top SASS instructions of one kernel in an ncu report (by executed count)."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ie = hdr.index('Instructions Executed')
ws = hdr.index('Warp Stall Sampling (All Samples)')
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ie] or 0), int(r[ws] or 0), r[0], r[1]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print('total warp-inst', tot)
ops = Counter()
for d in data:
    op = d[3].split()[0] if not d[3].strip().startswith('@') else d[3].split()[1]
    ops[op.split('.')[0]] += d[0]
print('by opcode:', ', '.join('%s %.1f%%' % (k, 100.0 * v / tot) for k, v in ops.most_common(25)))
mx = max(d[0] for d in data)
print('hottest-loop instructions (count == max %d):' % mx)
for d in data:
    if d[0] >= 0.9 * mx:
        print('  ', d[1], d[3][:100])
