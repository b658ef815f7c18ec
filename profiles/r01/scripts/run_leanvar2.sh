set -u
O=gpurun_out; mkdir -p $O
for v in "4,4" "4,5" "2,6" "6,4"; do
  for c in arxiv hyper; do
    RNN_LEAN_VAR=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${c}_lean2_$v.json 2>$O/bench_${c}_lean2_$v.err
  done
done
