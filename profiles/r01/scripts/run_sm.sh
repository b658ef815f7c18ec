# group-cached softmax walkers: parity under every instantiated variant, then MAG timing per variant
set -u
O=gpurun_out; mkdir -p $O
for v in "6,2,4,2" "4,3,2,3" "4,2,3,2" "8,2,4,2"; do
  RNN_SM_VAR=$v timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_sm_$v.log 2>&1; echo "exit $?" >> $O/pytest_sm_$v.log
done
RNN_SM_NOCACHE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax_small" -x -q > $O/pytest_sm_nocache.log 2>&1; echo "exit $?" >> $O/pytest_sm_nocache.log
timeout 900 python -m pytest tests/test_gpu_hgt_hyper.py -x -q > $O/pytest_hgt.log 2>&1; echo "exit $?" >> $O/pytest_hgt.log
RNN_SM_NOCACHE=1 timeout 600 python bench.py --config mag --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_nocache.json 2>$O/bench_mag_nocache.err
for v in "6,2,4,2" "4,3,2,3" "4,2,3,2" "8,2,4,2"; do
  RNN_SM_VAR=$v timeout 600 python bench.py --config mag --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_$v.json 2>$O/bench_mag_$v.err
done
