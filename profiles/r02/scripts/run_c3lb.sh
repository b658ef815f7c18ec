# load-balanced C3 (phase A/B long-list queue) + CTA-shape variants of C3 and C4, 0.1-scale products
set -u
O=gpurun_out/r02_c3lb; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x -k "not full_scale" > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
for v in base c3x256 c3x512 c4x512 c4x256 c4in4; do
  if [ $v = base ]; then unset RNN_LIB; else export RNN_LIB=$PWD/build/variants/librnn_$v.so; fi
  timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_$v.json 2> $O/dhn01_$v.err
done
export RNN_LIB=$PWD/build/variants/librnn_c4x256.so
RNN_DHN_COMPACT_IDS=1 timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_c4x256_compact.json 2> $O/dhn01_c4x256_compact.err
export RNN_LIB=$PWD/build/variants/librnn_c3x256.so
timeout 1200 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x -k "not full_scale" > $O/pytest_dhn_c3x256.log 2>&1; echo "exit $?" >> $O/pytest_dhn_c3x256.log
