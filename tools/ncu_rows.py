"""Top stall rows (SASS) of an ncu source page, optionally for one exec count (dev tool).
usage: python tools/ncu_rows.py report.ncu-rep [exec_count] [n]"""
import csv
import subprocess
import sys

out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si, ei = hdr.index('Source'), hdr.index('Instructions Executed')
ai = hdr.index('Address') if 'Address' in hdr else 0
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
want = int(sys.argv[2]) if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
sel = []
for r in rows[2:]:
    e = int(r[ei] or 0)
    if want is not None and e != want:
        continue
    st = {hdr[i][6:]: int(r[i] or 0) for i in stall_cols if int(r[i] or 0)}
    sel.append((sum(st.values()), r[ai], r[si].strip()[:60], st))
tot = sum(s[0] for s in sel)
print('total samples', tot)
for s in sorted(sel, key=lambda x: -x[0])[:n]:
    print(f'{s[0]:5d} {s[1]} {s[2]:60s} {dict(sorted(s[3].items(), key=lambda x: -x[1])[:3])}')
