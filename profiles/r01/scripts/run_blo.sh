set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -k "projection" -x -q > $O/pytest_blo.log 2>&1; echo "exit $?" >> $O/pytest_blo.log
timeout 300 python profiles/micro_dw.py > $O/micro_dw_blo.log 2>&1
RNN_NO_BLO=1 timeout 300 python profiles/micro_dw.py > $O/micro_dw_noblo.log 2>&1
timeout 600 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_blo.json 2>$O/bench_mag_blo.err
