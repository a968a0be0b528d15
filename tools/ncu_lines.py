"""Per-CUDA-source-line instruction and stall totals of one kernel in an ncu report.

    python tools/ncu_lines.py <rep> <kernel-regex> [top]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--kernel-name', 'regex:' + kern,
                      '--print-source', 'cuda,sass', '-c', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = []
cur_file = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        ie = hdr.index('Instructions Executed')
        ws = hdr.index('Warp Stall Sampling (All Samples)')
        continue
    if hdr and r and r[0] not in ('', '-') and len(r) > ie:
        try:
            res.append((int(r[ie] or 0), int(r[ws] or 0), cur_file, r[0], r[1][:90]))
        except ValueError:
            pass
tot = sum(x[0] for x in res)
tots = sum(x[1] for x in res)
print('total warp-inst %d, stall samples %d' % (tot, tots))
for x in sorted(res, reverse=True)[:top]:
    print('%5.1f%% %5.1f%%  %s:%s  %s' % (100.0 * x[0] / tot, 100.0 * x[1] / max(tots, 1), x[2], x[3], x[4]))
print('--- by stall samples')
for x in sorted(res, key=lambda r: -r[1])[:top]:
    print('%5.1f%% %5.1f%%  %s:%s  %s' % (100.0 * x[0] / tot, 100.0 * x[1] / max(tots, 1), x[2], x[3], x[4]))
