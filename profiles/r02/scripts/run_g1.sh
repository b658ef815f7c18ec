O=gpurun_out/r02_g1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
echo "new $(timeout 300 python profiles/r02/scripts/sweep_chunk.py 2>&1 | tail -1)" > $O/proj.txt
timeout 1200 python -m pytest tests/test_gpu_rgcn.py tests/test_gpu_select_stream.py tests/test_gpu_parity.py -q -k "not max_aggregate" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 1200 python -m pytest tests/test_gpu_full_scale.py -q > $O/pytest_full.log 2>&1; echo "exit $?" >> $O/pytest_full.log
timeout 600 python bench.py --config arxiv --seeds 42 --steps 10 --no-cpu-baseline --no-e2e > $O/arxiv.json 2> $O/arxiv.err
