#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
for f in 0 1 3; do for v in 0 1; do for w in C5 C2; do
 BDK_DEV_FLAGS=$f BDK_FAST_VARIANT=$v BDK_TRACE=gpurun_out/trace_${w}_v${v}_f$f.txt timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --soak 0 --steps 3 --warmup 3 > /dev/null 2>&1
done; done; done
echo done
