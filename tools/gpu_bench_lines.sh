#!/bin/bash
# bench.py lines of every workload (both arms for C2/C5/C4), no profilers:
# the bench_*.json set of tools/gpu_full.sh without the ncu passes.
mkdir -p gpurun_out/lines
O=gpurun_out/lines
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for w in C5 C3 C1 C2b4; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
for w in C4 C4b2; do timeout 600 python bench.py --workload $w --steps 100 > $O/bench_$w.json 2> $O/bench_$w.err; done
echo done
