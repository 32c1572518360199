#!/bin/bash
# Profiling pass: per-CTA timeline traces + ncu full captures (with source) of
# decode_fast for the given workloads (default C2 C5).
mkdir -p gpurun_out/${POUT:-prof}
O=gpurun_out/${POUT:-prof}
WL=${WL:-"C2 C5"}
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
for w in $WL; do
 rm -f $O/trace_$w.txt
 BDK_TRACE=$O/trace_$w.txt timeout 300 python bench.py --workload $w --quick --no-cpu-baseline --e2e-steps 0 --soak 0 --steps 3 --warmup 3 > /dev/null 2>&1
 python tools/trace_stats.py $O/trace_$w.txt > $O/trace_$w.stats 2>&1
 timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 8 -c 1 -f -o $O/prof_$w python bench.py --workload $w --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --quick --no-cpu-baseline > $O/ncu_full_$w.log 2>&1
done
echo done
