#!/bin/bash
# Knob sweep (dev): bench lines per (env setting, workload).  KNOBS is a list
# of "ENV=VAL" strings ("-" = defaults), WL a list of workloads.
mkdir -p gpurun_out/${KOUT:-knobs}
O=gpurun_out/${KOUT:-knobs}
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; fi
for k in ${KNOBS:--}; do for w in ${WL:-C2 C5}; do
  tag=$(echo "$k" | tr '=/' '__')
  if [ "$k" = "-" ]; then envs=""; else envs="$k"; fi
  env $envs timeout 300 python bench.py --workload $w --quick --no-cpu-baseline --e2e-steps ${E2E:-20} --soak 0.3 > $O/b_${w}_${tag}.json 2> $O/b_${w}_${tag}.err
  python - "$O/b_${w}_${tag}.json" "$k" "$w" >> $O/summary.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"{sys.argv[3]:3s} {sys.argv[2]:28s} value={d['value']:8.1f} frac={d['roofline']['frac']:.3f} us={d['latency_us']:7.2f} iso_us={d['roofline'].get('kernel_isolated_us') or 0:7.2f} e2e={e.get('value')} e2e_us={e.get('latency_us')}")
except Exception as ex:
    print(sys.argv[3], sys.argv[2], "FAILED", ex)
PY
done; done
cat $O/summary.txt
