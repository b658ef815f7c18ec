O=gpurun_out/r02_prec; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python profiles/r02/scripts/dbg_prec.py > $O/prec_after.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "projection" > $O/proj_parity.log 2>&1
timeout 900 python -m pytest tests/test_gpu_full_scale.py tests/test_gpu_programs.py tests/test_gpu_hgt_hyper.py -q -x --durations=5 > $O/full.log 2>&1
timeout 900 python bench.py --config mag --steps 10 --warmup 3 --seeds 42 --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 900 python bench.py --config hyper --steps 10 --warmup 3 --seeds 42 --no-cpu-baseline > $O/bench_hyper.json 2> $O/bench_hyper.err
timeout 900 python bench.py --config arxiv --steps 10 --warmup 3 --seeds 42 --no-cpu-baseline > $O/bench_arxiv.json 2> $O/bench_arxiv.err
