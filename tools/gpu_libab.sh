#!/bin/bash
# A/B of library builds (dev): bench lines with BDK_LIB=<each .so in LIBS>
# ("-" = the in-tree build), interleaved over ROUNDS passes.
mkdir -p gpurun_out/libab
O=gpurun_out/libab
: > $O/summary.txt
for r in $(seq ${ROUNDS:-2}); do
for l in ${LIBS:--}; do for w in ${WL:-C5 C2 C1}; do
  tag=$(basename $l .so)
  if [ "$l" = "-" ]; then envs=""; tag=intree; else envs="BDK_LIB=$l"; fi
  env $envs timeout 300 python bench.py --workload $w --quick --no-cpu-baseline --e2e-steps ${E2E:-20} --soak 0.3 ${EXTRA} > $O/b_${w}_${tag}_$r.json 2> $O/b_${w}_${tag}_$r.err
  python - "$O/b_${w}_${tag}_$r.json" "$tag" "$w" >> $O/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"{sys.argv[3]:4s} {sys.argv[2]:12s} value={d['value']:8.1f} frac={d['roofline']['frac']:.3f} us={d['latency_us']:7.2f} iso_us={d['roofline'].get('kernel_isolated_us') or 0:7.2f} e2e={e.get('value')} e2e_us={e.get('latency_us')}")
except Exception as ex:
    print(sys.argv[3], sys.argv[2], "FAILED", ex)
PY
done; done; done
cat $O/summary.txt
