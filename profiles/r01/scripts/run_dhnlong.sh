set -u
O=gpurun_out; mkdir -p $O
for v in long48 long256; do
  RNN_LIB=build/variants/librnn_$v.so timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_$v.json 2> $O/bench_dhn_$v.err
done
RNN_LIB=build/variants/librnn_long48.so timeout 900 python -m pytest tests/test_gpu_dhn.py -x -q -k "products or symmetric" > $O/pytest_dhn_long48.log 2>&1; echo "exit $?" >> $O/pytest_dhn_long48.log
