#!/bin/bash
# Round-2 measurement pass on one B200: parity tests, smoke, bench (default
# line with extras + parity, per-workload lines, reference arm), flush-step
# latency, trace stats, ncu launch list + full captures of the hot kernels,
# and steady-state (application replay, no cache flush) DRAM bytes per launch.
O=gpurun_out/${OUT:-r02}; mkdir -p $O

python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
nvidia-smi -L > $O/gpu.txt 2>&1; lscpu > $O/host_cpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in C5 C2 C3 C1 C2b4; do timeout 600 python bench.py --workload $w --quick --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:combine_fast -s 8 -c 1 -f -o /tmp/prof_cmb python bench.py --workload C5 --quick --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full_combine_C5.log 2>&1
python tools/ncu_summary.py /tmp/prof_cmb.ncu-rep > $O/ncu_summary_combine_C5.txt 2>&1
for w in C4 C4b2; do timeout 600 python bench.py --workload $w --quick --steps 100 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --impl reference > $O/bench_ref_C5.json 2> $O/bench_ref_C5.err
python tools/flush_step.py C5 C2 C3 C1 > $O/flush_step.txt 2>&1
python tools/trace_run.py C5 /tmp/tr_c5.txt 10 > /dev/null 2>&1; python tools/trace_stats.py /tmp/tr_c5.txt > $O/trace_stats_C5.txt; python tools/trace_sm.py /tmp/tr_c5.txt > $O/trace_sm_C5.txt
python tools/trace_run.py C2 /tmp/tr_c2.txt 10 > /dev/null 2>&1; python tools/trace_stats.py /tmp/tr_c2.txt > $O/trace_stats_C2.txt; python tools/trace_sm.py /tmp/tr_c2.txt > $O/trace_sm_C2.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --quick --steps 20 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# steady state: application replay, caches not flushed -> DRAM bytes of one launch inside the loop
for w in C5 C2; do
timeout 900 ncu --replay-mode application --cache-control none --clock-control none -k regex:decode_fast -s 30 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum --csv python bench.py --workload $w --quick --steps 40 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_steady_$w.csv 2> $O/ncu_steady_$w.err
done
for w in C5 C2 C3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 8 -c 1 -f -o /tmp/prof_$w python bench.py --workload $w --quick --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full_$w.log 2>&1
python tools/ncu_summary.py /tmp/prof_$w.ncu-rep > $O/ncu_summary_$w.txt 2>&1
python tools/ncu_mix.py /tmp/prof_$w.ncu-rep > $O/ncu_mix_$w.txt 2>&1
done
for w in C4 C4b2; do
timeout 900 ncu --set full --metrics lts__t_sectors_op_write.sum --clock-control none --import-source on -k regex:qpack_fast -s 5 -c 1 -f -o /tmp/prof_$w python bench.py --workload $w --quick --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_$w.log 2>&1
python tools/ncu_summary.py /tmp/prof_$w.ncu-rep > $O/ncu_summary_$w.txt 2>&1
python tools/ncu_mix.py /tmp/prof_$w.ncu-rep > $O/ncu_mix_$w.txt 2>&1
done
du -sh $O
echo done
