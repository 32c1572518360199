#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in C2 C5 C1 C3; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --e2e-steps 10 --soak 0.3 > gpurun_out/bench_${w}.json 2> gpurun_out/bench_${w}.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 6 -c 1 -o gpurun_out/prof_c5 python bench.py --workload C5 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 6 -c 1 -o gpurun_out/prof_c2 python bench.py --workload C2 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
echo done
