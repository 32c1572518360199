#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for p in 1 0; do for w in C2 C5 C3 C1; do BDK_PDL=$p timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --soak 0.3 > gpurun_out/bench_${w}_p$p.json 2> gpurun_out/bench_${w}_p$p.err; done; done
echo done
