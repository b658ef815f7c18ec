# lean (GCN / hypergraph) gather-reduce variants: rows in flight U, min CTAs per SM
set -u
O=gpurun_out; mkdir -p $O
for v in "8,0" "4,4" "8,4" "8,3" "4,6"; do
  for c in arxiv hyper; do
    RNN_LEAN_VAR=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_${c}_lean_$v.json 2>$O/bench_${c}_lean_$v.err
  done
done
RNN_LEAN_VAR="4,6" timeout 900 python -m pytest tests/test_gpu_parity.py -k "fwd_bwd" -x -q > $O/pytest_lean.log 2>&1; echo "exit $?" >> $O/pytest_lean.log
