set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_programs.py tests/test_gpu_hgt_hyper.py tests/test_gpu_shard.py -x -q > $O/pytest_last2.log 2>&1; echo "pytest exit $?" >> $O/pytest_last2.log
timeout 600 python bench.py > $O/bench_arxiv.json 2> $O/bench_arxiv.err
timeout 900 python bench.py --config hyper --steps 10 --warmup 3 > $O/bench_hyper.json 2> $O/bench_hyper.err
timeout 900 python bench.py --config cora --steps 10 --warmup 3 > $O/bench_cora.json 2> $O/bench_cora.err
