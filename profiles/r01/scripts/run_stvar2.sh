set -u
O=gpurun_out; mkdir -p $O
RNN_ST_VAR="4,3,1,5,2,4" timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_st15.log 2>&1; echo "exit $?" >> $O/pytest_st15.log
for v in "4,3,1,4,2,4" "4,3,1,5,2,4" "1,5,1,5,2,4"; do
  RNN_ST_VAR=$v timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_st_$v.json 2>$O/bench_mag_st_$v.err
done
