"""Per-SM loop-time consistency across traced launches (dev tool).

python tools/trace_sm.py TRACE.txt
For each launch: per-CTA packed-loop time (stamps 1 -> 2); per SM the mean of
its CTAs.  Prints the spread, the correlation of per-SM times between
launches (systematic vs random slow SMs), and the step time a perfectly
balanced split of the same total loop work would give.
"""
import sys

import numpy as np

launches = open(sys.argv[1]).read().split("launch ")[1:]
per_sm = []
for L in launches:
    rows = L.strip().splitlines()[1:]
    a = np.array([[int(x) for x in r.split()] for r in rows], dtype=np.float64)
    a = a[(a[:, 0] > 0) & (a[:, 1] > 0)]
    t0 = a[:, 0].min()
    loop = (a[:, 2] - a[:, 1]) / 1e3
    end = (a[:, 5] - t0) / 1e3
    first = (a[:, 1] - t0) / 1e3
    sm = a[:, 8].astype(int)
    v = np.zeros(148)
    c = np.zeros(148)
    for s, l in zip(sm, loop):
        v[s] += l
        c[s] += 1
    v = np.where(c > 0, v / np.maximum(c, 1), np.nan)
    per_sm.append(v)
    print(f"loop us p0 {loop.min():6.2f} p50 {np.median(loop):6.2f} p100 {loop.max():6.2f} | "
          f"first block p50 {np.median(first):5.2f} max {first.max():5.2f} | end max {end.max():6.2f} "
          f"| balanced loop {loop.mean():6.2f}")
P = np.array(per_sm)
ok = ~np.isnan(P).any(axis=0)
P = P[:, ok]
if len(P) > 2:
    cc = np.corrcoef(P)
    iu = np.triu_indices(len(P), 1)
    print(f"per-SM loop time correlation between launches: mean {cc[iu].mean():.2f} "
          f"(1 = the same SMs are slow every launch)")
    m = P.mean(axis=0)
    order = np.argsort(m)
    print("slowest SMs (mean loop us):", [(int(np.nonzero(ok)[0][i]), round(m[i], 2)) for i in order[-8:]])
    print("fastest SMs:", [(int(np.nonzero(ok)[0][i]), round(m[i], 2)) for i in order[:8]])
