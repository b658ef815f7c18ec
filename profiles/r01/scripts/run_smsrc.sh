# source-major softmax backward (D, pass A, pass B) vs the two-pass (a, de) scheme
set -u
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -k "softmax" -x -q > $O/pytest_smsrc.log 2>&1; echo "exit $?" >> $O/pytest_smsrc.log
timeout 900 python -m pytest tests/test_gpu_hgt_hyper.py tests/test_gpu_shard.py -x -q > $O/pytest_smsrc_prog.log 2>&1; echo "exit $?" >> $O/pytest_smsrc_prog.log
RNN_SM_TWOPASS=1 timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_twopass.json 2>$O/bench_mag_twopass.err
for v in "4,3,1,4,2,4" "4,3,2,3,4,3" "4,3,1,4,4,3" "4,3,2,4,4,3"; do
  RNN_ST_VAR=$v timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_src_$v.json 2>$O/bench_mag_src_$v.err
done
