O=gpurun_out/r02_f12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "epilogue or max_aggregate or empty_join or projection" > $O/pytest_parity.log 2>&1; echo "exit $?" >> $O/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_shard.py -q -x > $O/pytest_prog.log 2>&1; echo "exit $?" >> $O/pytest_prog.log
timeout 600 python -m pytest tests/test_gpu_dhn.py -q -x -k "root_subset or symmetry" > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 900 python bench.py --config mag --seeds 42 --steps 10 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 900 python bench.py --config arxiv --seeds 42 --steps 10 --no-cpu-baseline > $O/bench_arxiv.json 2> $O/bench_arxiv.err
