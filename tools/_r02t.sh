set -x
O=gpurun_out/r02t
mkdir -p $O
timeout 900 python bench.py --config c2h --no-cpu-baseline --budget-scale 1.5 > $O/bench_c2h_b15.json 2> $O/bench_c2h_b15.err
timeout 900 python bench.py --config c2h --no-cpu-baseline --budget-scale 1.25 > $O/bench_c2h_b125.json 2> $O/bench_c2h_b125.err
for w in 1 2 4 8; do
  timeout 900 python bench.py --config c4s --workers $w --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_c4s_w$w.json 2> $O/bench_c4s_w$w.err
done
