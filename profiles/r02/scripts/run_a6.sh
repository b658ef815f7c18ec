set -u
O=gpurun_out/r02_a6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dhn_scale.py -q --durations=15 > $O/pytest_dhn_scale.log 2>&1; echo "pytest exit $?" >> $O/pytest_dhn_scale.log
timeout 1200 python -m pytest tests/test_gpu_full_scale.py tests/test_gpu_hgt_hyper.py tests/test_gpu_shard.py tests/test_gpu_dhn.py tests/test_gpu_parity.py -q --durations=8 > $O/pytest_full.log 2>&1; echo "pytest exit $?" >> $O/pytest_full.log
timeout 900 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
