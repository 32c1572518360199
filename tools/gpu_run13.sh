#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
for w in C5 C2 C3; do
 BDK_TRACE=gpurun_out/trace_${w}.txt timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --soak 0 --steps 3 --warmup 3 > /dev/null 2>&1
done
echo done
