#!/bin/bash
# One gpurun session: parity tests, smoke, bench lines, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1; nvidia-smi -q | grep -i -E "product name|l2|clocks" | head -20 >> gpurun_out/gpu.txt
lscpu | head -20 > gpurun_out/host_cpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --workload C5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --workload C3 --no-cpu-baseline --steps 50 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --workload C1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 6 -c 2 -o gpurun_out/prof_c2 python bench.py --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 6 -c 2 -o gpurun_out/prof_c5 python bench.py --workload C5 --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_c5.log 2>&1
echo done
