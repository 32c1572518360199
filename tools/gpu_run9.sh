#!/bin/bash
mkdir -p gpurun_out
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 6 -c 1 -o gpurun_out/prof_c5_v0 python bench.py --workload C5 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c5_v0.log 2>&1
BDK_FAST_VARIANT=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 6 -c 1 -o gpurun_out/prof_c5_v1 python bench.py --workload C5 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c5_v1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 6 -c 1 -o gpurun_out/prof_c2_v0 python bench.py --workload C2 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_c2_v0.log 2>&1
echo done
