# the walk code of c47154b (no prefetch / probe / per-root table switches): DHN parity, benches
set -u
O=gpurun_out/r02_dhn47; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/dhn01.json 2> $O/dhn01.err
timeout 1500 python bench.py --config dhn --steps 2 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
