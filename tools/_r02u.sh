set -x
O=gpurun_out/r02u
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
LAIVG_TRACE=1 ONLY=4096 MODES=fused timeout 300 python tools/fused_probe.py > $O/trace.jsonl 2> $O/trace.err
