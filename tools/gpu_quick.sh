#!/bin/bash
# Quick pass: GPU parity tests + bench lines for the main workloads.
mkdir -p gpurun_out/quick
O=gpurun_out/quick
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in C2 C5 C3 C1; do timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 > $O/bench_${w}.json 2> $O/bench_${w}.err; done
echo done
