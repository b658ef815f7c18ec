set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dhn.py -x -q > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 900 python -m pytest tests/test_gpu_parity.py -k "projection" -x -q > $O/pytest_proj.log 2>&1; echo "exit $?" >> $O/pytest_proj.log
timeout 900 python -m pytest tests/test_gpu_hgt_hyper.py tests/test_gpu_programs.py -x -q > $O/pytest_prog.log 2>&1; echo "exit $?" >> $O/pytest_prog.log
timeout 900 python bench.py --config mag --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_mag_new.json 2> $O/bench_mag_new.err
timeout 900 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn_new.json 2> $O/bench_dhn_new.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_arxiv_new.json 2> $O/bench_arxiv_new.err
