#!/bin/bash
# GPU pass: selected pytest files (args, default all gpu tests) + the default
# bench line as the driver runs it.  Outputs under gpurun_out/$OUT.
OUT=${OUT:-check}
mkdir -p gpurun_out/$OUT
O=gpurun_out/$OUT
python -c "from paper_2503_18773_b200 import build as B; assert not B._stale(), \"stale lib\"" || exit 3
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi_before.txt 2>&1
timeout 1500 python -m pytest ${TESTS:-tests} -m gpu -x -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
  echo "bench rc=$?" >> $O/bench.err
fi
echo done
