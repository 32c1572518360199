#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
for v in 3 0 1; do for w in C2 C5 C3; do BDK_FAST_VARIANT=$v timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --soak 0.3 > gpurun_out/bench_${w}_v$v.json 2> gpurun_out/bench_${w}_v$v.err; done; done
BDK_FAST_VARIANT=3 BDK_TRACE=gpurun_out/trace_C5v3.txt timeout 300 python bench.py --workload C5 --no-cpu-baseline --e2e-steps 0 --soak 0 --steps 3 --warmup 3 > /dev/null 2>&1
BDK_FAST_VARIANT=3 timeout 600 python -m pytest tests -m gpu -x -q -k "decode" > gpurun_out/pytest_v3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v3.log
echo done
