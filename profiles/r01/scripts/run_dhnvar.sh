# DHN C4 CTA-shape variants (threads per root CTA x CTAs per SM, table slots)
set -u
O=gpurun_out; mkdir -p $O
for v in dhn512x2 dhn256x4 dhn1024c8k; do
  L=build/variants/librnn_$v.so
  RNN_LIB=$L timeout 900 python -m pytest tests/test_gpu_dhn.py -x -q -k "random or ragged or products" > $O/pytest_$v.log 2>&1; echo "exit $?" >> $O/pytest_$v.log
  RNN_LIB=$L timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_$v.json 2> $O/bench_dhn_$v.err
done
