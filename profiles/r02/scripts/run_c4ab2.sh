# C4 slot walk without the prefetch smem: partition probe on / off; DHN tests; full-scale bench
set -u
O=gpurun_out/r02_c4ab2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/dhn01_$1.json 2> $O/dhn01_$1.err; }
run default
RNN_DHN_NO_PROBE=1 run noprobe
RNN_DHN_PREFETCH=1 RNN_DHN_NO_PROBE=1 run prefetch_noprobe
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 1500 python bench.py --config dhn --steps 2 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
