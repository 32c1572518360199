"""Per-role / per-opcode stall attribution from an ncu source page (dev tool).
usage: python tools/ncu_src.py report.ncu-rep [exec_count_filter]"""
import collections
import csv
import subprocess
import sys

path = sys.argv[1]
out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
si, ei = hdr.index('Source'), hdr.index('Instructions Executed')
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
byexec = collections.defaultdict(lambda: collections.Counter())
byop = collections.defaultdict(lambda: collections.Counter())
for r in data:
    e = int(r[ei] or 0)
    src = r[si].strip().split()
    op = src[1] if src and src[0].startswith('@') else (src[0] if src else '?')
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            byexec[e][hdr[i]] += v
            byop[op.split('.')[0]][hdr[i]] += v
filt = int(sys.argv[2]) if len(sys.argv) > 2 else None
print('== by execution count (role proxy)')
for e, c in sorted(byexec.items(), key=lambda x: -sum(x[1].values()))[:8]:
    print(e, sum(c.values()), dict(c.most_common(6)))
print('== by opcode')
for op, c in sorted(byop.items(), key=lambda x: -sum(x[1].values()))[:20]:
    print(f'{op:10s}', sum(c.values()), dict(c.most_common(4)))
