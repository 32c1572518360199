#!/bin/bash
# Full measurement pass on one B200: parity tests, smoke, bench lines (all
# workloads, both arms), ncu launch list + full captures of the hot kernels.
mkdir -p gpurun_out/full
O=gpurun_out/full
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
nvidia-smi -L > $O/gpu.txt 2>&1; lscpu > $O/host_cpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for w in C5 C3 C1 C2b4; do timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
for w in C4 C4b2; do timeout 600 python bench.py --workload $w --steps 100 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
timeout 900 python bench.py --impl reference --workload C5 --steps 3 --warmup 1 > $O/bench_ref_C5.json 2> $O/bench_ref_C5.err
timeout 900 python bench.py --impl reference --workload C4 > $O/bench_ref_C4.json 2> $O/bench_ref_C4.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv python bench.py --steps 20 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1
# full captures: summarized on the box (the .ncu-rep files stay there; the
# 64 MiB gpurun_out cap would drop everything)
for w in C2 C5 C3; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 8 -c 1 -f -o /tmp/prof_$w python bench.py --workload $w --steps 5 --warmup 3 --soak 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full_$w.log 2>&1
python tools/ncu_summary.py /tmp/prof_$w.ncu-rep > $O/ncu_summary_$w.txt 2>&1
ncu -i /tmp/prof_$w.ncu-rep --page details --csv > $O/ncu_details_$w.csv 2>/dev/null
python tools/ncu_mix.py /tmp/prof_$w.ncu-rep > $O/ncu_mix_$w.txt 2>&1
done
for w in C4 C4b2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qpack_fast -s 5 -c 1 -f -o /tmp/prof_$w python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/ncu_full_$w.log 2>&1
python tools/ncu_summary.py /tmp/prof_$w.ncu-rep > $O/ncu_summary_$w.txt 2>&1
ncu -i /tmp/prof_$w.ncu-rep --page details --csv > $O/ncu_details_$w.csv 2>/dev/null
python tools/ncu_mix.py /tmp/prof_$w.ncu-rep > $O/ncu_mix_$w.txt 2>&1
done
du -sh $O
echo done
