#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in C5 C2 C3; do
 BDK_TRACE=gpurun_out/trace_${w}.txt timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 0 --soak 0 --steps 3 --warmup 3 > /dev/null 2>&1
done
for w in C2 C5 C3 C1; do timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --soak 0.3 > gpurun_out/bench_${w}.json 2> gpurun_out/bench_${w}.err; done
echo done
