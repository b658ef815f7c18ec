O=gpurun_out/r02_f3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "epilogue or max_aggregate" > $O/pytest_parity.log 2>&1; echo "exit $?" >> $O/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_programs.py -q > $O/pytest_train.log 2>&1; echo "exit $?" >> $O/pytest_train.log
timeout 900 python bench.py --config arxiv --seeds 42 --steps 10 --no-cpu-baseline > $O/bench_arxiv.json 2> $O/bench_arxiv.err
timeout 900 python bench.py --config cora --seeds 42 --steps 20 --no-cpu-baseline > $O/bench_cora.json 2> $O/bench_cora.err
for ch in 256 1024 4096; do echo $ch; done > /dev/null
timeout 900 python bench.py --config mag --seeds 42 --steps 10 --no-cpu-baseline --no-e2e > $O/bench_mag.json 2> $O/bench_mag.err
