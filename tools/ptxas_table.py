"""ptxas -v resource table of the fast decode kernels (dev tool).

python tools/ptxas_table.py [file.cu] [filter]
"""
import re
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "paper_2503_18773_b200/csrc/bdk_decode_fast.cu"
flt = sys.argv[2] if len(sys.argv) > 2 else "decode_fast_kernel"
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "--expt-relaxed-constexpr", "-diag-suppress", "177", "-Xptxas", "-v", "-c", src,
                      "-o", "/tmp/_ptxas_table.o"], capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None or flt not in cur:
        continue
    short = re.search(r"kernel(I\S+?)EEEv", cur)
    key = short.group(1) if short else cur
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(key, {}).update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(key, {})["regs"] = int(m.group(1))
for k in sorted(rows):
    r = rows[k]
    print(f"{k:40s} regs {r.get('regs')}  stack {r.get('stack')}  spill st/ld {r.get('st')}/{r.get('ld')}")
if "error" in out:
    print(out)
