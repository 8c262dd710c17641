#!/bin/bash
# One GPU session: gpu tests, smoke, bench (C2, C1, c2b), launch lists, full ncu
# of the dominant kernel (fused_query_kernel on the single-query path).
# usage (from repo root, under gpurun): bash tools/gpu_check.sh [tag]
set -x
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
if [ "${TESTS:-1}" = 1 ]; then
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 900 python bench.py --config c2b --steps 5 --warmup 3 > $O/bench_c2b.json 2> $O/bench_c2b.err
if [ "${NCU:-1}" = 1 ]; then
for cfg in c2 c1; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_$cfg.csv python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch_$cfg.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_query -s 6 -c 2 \
  -o $O/fused_full_$cfg python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full_$cfg.log 2>&1
done
fi
