set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dhn.py -x -q > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_sym.json 2> $O/bench_dhn_sym.err
