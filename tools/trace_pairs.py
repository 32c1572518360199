import sys, numpy as np, collections
lines = open(sys.argv[1]).read().split("launch ")[1:]
blk = lines[-2].strip().splitlines()
a = np.array([[int(x) for x in l.split()] for l in blk[1:]], dtype=np.float64)
a = a[a[:, 0] > 0]
loop_end = (a[:, 2] - a[:, 0].min()) / 1e3
loop = (a[:, 2] - a[:, 1]) / 1e3
sm = a[:, 8].astype(int)
d = collections.defaultdict(list)
for i in range(len(a)):
    d[sm[i]].append((loop[i], loop_end[i]))
diffs = []; ends = []; smmax = []
for s, v in d.items():
    if len(v) == 2:
        diffs.append(abs(v[0][0] - v[1][0])); smmax.append(max(v[0][1], v[1][1]))
print("SMs with 2 CTAs:", len(diffs), "pair |loop diff| p50/p90/max", np.percentile(diffs, [50, 90, 100]).round(2))
print("per-SM finish (max of pair) p10/p50/p90/max", np.percentile(smmax, [10, 50, 90, 100]).round(2))
print("CTA loop p10/p50/p90/max", np.percentile(loop, [10, 50, 90, 100]).round(2))
# within an SM pair: is the faster CTA the one that started first / has the lower blockIdx?
first_faster = lower_faster = n = 0
idx = {}
for i in range(len(a)):
    idx.setdefault(sm[i], []).append(i)
for s, v in idx.items():
    if len(v) != 2:
        continue
    i, j = v
    fast, slow = (i, j) if loop[i] < loop[j] else (j, i)
    n += 1
    first_faster += a[fast, 0] <= a[slow, 0]
    lower_faster += fast < slow
print(f"pairs {n}: faster CTA started first in {first_faster}, has lower blockIdx in {lower_faster}")
