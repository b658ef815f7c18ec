# full table for every root (default again) with the probe off: DHN parity + full-scale bench
set -u
O=gpurun_out/r02_dhnlast; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 1500 python bench.py --config dhn --steps 2 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
RNN_DHN_ROOT_TABLE=1 timeout 1500 python bench.py --config dhn --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_dhn_roottable.json 2> $O/bench_dhn_roottable.err
