set -x
O=gpurun_out/r02v
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_batch.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
ENTRIES=host MODES=fused,fused timeout 300 python tools/fused_probe.py > $O/wc.jsonl 2>/dev/null
LAIVG_HQ_NOWC=1 ENTRIES=host MODES=fused,fused timeout 300 python tools/fused_probe.py > $O/nowc.jsonl 2>/dev/null
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
