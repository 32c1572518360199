"""Per-opcode instruction counts of the rows executed N times (dev tool).
usage: python tools/ncu_mix.py report.ncu-rep [min_exec]"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si, ei = hdr.index('Source'), hdr.index('Instructions Executed')
byexec = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    e = int(r[ei] or 0)
    src = r[si].strip().split()
    op = src[1] if src and src[0].startswith('@') else (src[0] if src else '?')
    byexec[e][op.split('.')[0]] += 1
tot = collections.Counter()
for e, c in byexec.items():
    for op, n in c.items():
        tot[op] += n * e
print('total warp-inst', sum(tot.values()))
for e, c in sorted(byexec.items(), key=lambda x: -x[0] * sum(x[1].values()))[:8]:
    print(f'exec={e} rows={sum(c.values())} share={e*sum(c.values())/sum(tot.values()):.3f}', dict(c.most_common(14)))
