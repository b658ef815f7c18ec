# relu-fused projection fix (arxiv) + C3 CTA-shape variants (used-slot clear) at 0.1 scale
set -u
O=gpurun_out/r02_c3var; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python profiles/r02/scripts/probe_relu.py > $O/probe_relu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "relu" > $O/pytest_relu.log 2>&1; echo "exit $?" >> $O/pytest_relu.log
timeout 900 python bench.py --config arxiv --no-cpu-baseline > $O/bench_arxiv.json 2> $O/bench_arxiv.err
for v in base c3x512 c3x256 c4in4; do
  if [ $v = base ]; then unset RNN_LIB; else export RNN_LIB=$PWD/build/variants/librnn_$v.so; fi
  timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_$v.json 2> $O/dhn01_$v.err
done
unset RNN_LIB
export RNN_LIB=$PWD/build/variants/librnn_c3x512.so
timeout 900 python -m pytest tests/test_gpu_dhn.py -q -x -k "not products and not program" > $O/pytest_dhn_c3x512.log 2>&1; echo "exit $?" >> $O/pytest_dhn_c3x512.log
