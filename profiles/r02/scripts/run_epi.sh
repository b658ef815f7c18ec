# bias-only epilogue backward fast path: epilogue / program parity, arxiv + cora benches
set -u
O=gpurun_out/r02_epi; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_programs.py tests/test_gpu_train.py tests/test_gpu_shard.py -q -x -k "epi or gcn or program or train or shard or relu" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --config arxiv > $O/bench_arxiv.json 2> $O/bench_arxiv.err
timeout 900 python bench.py --config cora > $O/bench_cora.json 2> $O/bench_cora.err
