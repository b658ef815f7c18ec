set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dhn.py -x -q > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
RNN_DHN_SCALAR=1 timeout 900 python -m pytest tests/test_gpu_dhn.py -x -q -k "ragged or products" > $O/pytest_dhn_scalar.log 2>&1; echo "exit $?" >> $O/pytest_dhn_scalar.log
timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_v4.json 2> $O/bench_dhn_v4.err
RNN_DHN_SCALAR=1 timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_scalar.json 2> $O/bench_dhn_scalar.err
