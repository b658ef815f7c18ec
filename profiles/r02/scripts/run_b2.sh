O=gpurun_out/r02_b2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_shard.py -q --durations=5 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1200 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
timeout 900 python bench.py --config hyper --seeds 42 --no-cpu-baseline > $O/bench_hyper.json 2> $O/bench_hyper.err
timeout 1500 python bench.py --config dhn --steps 3 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
