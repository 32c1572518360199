"""Summarize BDK_TRACE output (per-CTA globaltimer stamps) of the last launch."""
import sys

import numpy as np

lines = open(sys.argv[1]).read().split("launch ")[1:]
which = int(sys.argv[2]) if len(sys.argv) > 2 else -1
blk = lines[which].strip().splitlines()
print(blk[0])
a = np.array([[int(x) for x in l.split()] for l in blk[1:]], dtype=np.float64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
def q(x):
    return " ".join(f"{np.percentile(x, p):8.2f}" for p in (0, 10, 50, 90, 100))
print("                     min      p10      p50      p90      max  (us)")
print("start            ", q((a[:, 0] - t0) / 1e3))
has1 = a[:, 1] > 0
print("first block ready", q((a[has1, 1] - a[has1, 0]) / 1e3))
print("packed loop      ", q((a[has1, 2] - a[has1, 1]) / 1e3))
print("residual         ", q((a[:, 3] - a[:, 2]) / 1e3))
print("finalize         ", q((a[:, 4] - a[:, 3]) / 1e3))
print("atomic+merge     ", q((a[:, 5] - a[:, 4]) / 1e3))
print("end (abs)        ", q((a[:, 5] - t0) / 1e3))
m = a[:, 6] > 0
if m.any():  # round-1 in-kernel merge stamps (the combine grid has none)
    print("merge (last CTAs)", q((a[m, 5] - a[m, 4]) / 1e3), "n=", m.sum())
if m.any() and a.shape[1] > 10 and (a[m, 10] > 0).all():
    print("  of which atomic ", q((a[m, 10] - a[m, 4]) / 1e3))
    print("  merge_cell      ", q((a[m, 5] - a[m, 10]) / 1e3))
    m2 = m & (a[:, 14] > 0) & (a[:, 15] > 0)  # merge_cell stamps (merge_cell_few has none)
    if m2.any():
        print("    ml loads      ", q((a[m2, 14] - a[m2, 10]) / 1e3), "n=", m2.sum())
        print("    weights+o     ", q((a[m2, 15] - a[m2, 14]) / 1e3))
        print("    rest          ", q((a[m2, 5] - a[m2, 15]) / 1e3))
    print("  merge end (abs) ", q((a[m, 5] - t0) / 1e3))
    print("  loop end of last", q((a[m, 2] - t0) / 1e3))
print("units/CTA", q(a[:, 7]))
if a.shape[1] > 9:
    print("cons. wait (ns->us)", q(a[:, 9] / 1e3))
    print("TMA empty-wait   ", q(a[:, 11] / 1e3))
    print("prep full-wait   ", q(a[:, 12] / 1e3))
    print("prep busy        ", q(a[:, 13] / 1e3))
    loop = (a[:, 2] - a[:, 1]) / 1e3
    # per-SM: both CTAs on an SM
    sm = a[:, 8].astype(int)
    order = np.argsort(loop)
    print("slowest CTAs (blk, sm, loop us, wait us):")
    for i in order[-6:]:
        print("   ", i, sm[i], round(loop[i], 2), round(a[i, 9] / 1e3, 2))
    print("fastest:")
    for i in order[:4]:
        print("   ", i, sm[i], round(loop[i], 2), round(a[i, 9] / 1e3, 2))
    import collections
    cnt = collections.Counter(sm)
    print("CTAs per SM histogram", collections.Counter(cnt.values()))
