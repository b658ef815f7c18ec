set -u
O=gpurun_out; mkdir -p $O
RNN_ST_VAR="4,3,1,4,4,4" timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_passb.log 2>&1; echo "exit $?" >> $O/pytest_passb.log
for v in "4,3,1,4,2,4" "4,3,1,4,4,4" "4,3,1,4,8,4"; do
  RNN_ST_VAR=$v timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_pb_$v.json 2>$O/bench_mag_pb_$v.err
done
