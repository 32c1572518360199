#!/bin/bash
# A/B of builds (dev): bench lines of each worktree under abtest/ plus the
# current tree, interleaved (ROUNDS passes) so box drift hits every build.
mkdir -p gpurun_out/ab
O=gpurun_out/ab
: > $O/summary.txt
for r in $(seq ${ROUNDS:-2}); do
for d in ${DIRS:-abtest/* .}; do for w in ${WL:-C5 C2 C1}; do
  tag=$(basename $(realpath $d))
  extra="--no-cpu-baseline"
  grep -q -- "--quick" $d/bench.py && extra="--quick --no-cpu-baseline"
  (cd $d && timeout 300 python bench.py --workload $w $extra --e2e-steps 20 --soak 0.3) > $O/b_${w}_${tag}_$r.json 2> $O/b_${w}_${tag}_$r.err
  python - "$O/b_${w}_${tag}_$r.json" "$tag" "$w" >> $O/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"{sys.argv[3]:4s} {sys.argv[2]:10s} value={d['value']:8.1f} frac={d['roofline']['frac']:.3f} us={d.get('latency_us', d.get('ms_per_step',0)*1e3):7.2f} iso_us={d['roofline'].get('kernel_isolated_us') or 0:7.2f} e2e={e.get('value')} e2e_us={e.get('latency_us')}")
except Exception as ex:
    print(sys.argv[3], sys.argv[2], "FAILED", ex)
PY
done; done; done
cat $O/summary.txt
