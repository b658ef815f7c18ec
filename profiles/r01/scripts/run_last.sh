set -u
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
RNN_ST_VAR="4,4,1,4,4,4" timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_f44.json 2>$O/bench_mag_f44.err
timeout 600 python bench.py > $O/bench_arxiv.json 2> $O/bench_arxiv.err
for c in cora hyper mag; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --config dhn --steps 3 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
