# softmax walker variants (rows in flight U, min CTAs/SM) on the full MAG step
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_st.log 2>&1; echo "exit $?" >> $O/pytest_st.log
for v in "2,4,1,4,2,4" "2,4,2,3,1,4" "1,4,1,4,1,4" "4,3,1,4,4,3"; do
  RNN_ST_VAR=$v timeout 600 python bench.py --config mag --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_st_$v.json 2>$O/bench_mag_st_$v.err
done
RNN_ST_VAR="2,4,1,4,2,4" timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_st2.log 2>&1; echo "exit $?" >> $O/pytest_st2.log
