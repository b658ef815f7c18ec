# projection rework check: tf32 conversion probe, projection parity, program parity, benches
set -u
O=gpurun_out; mkdir -p $O
timeout 300 python profiles/probe_tf32.py > $O/probe_tf32.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "projection" -x -q > $O/pytest_proj.log 2>&1; echo "exit $?" >> $O/pytest_proj.log
timeout 900 python -m pytest tests/test_gpu_programs.py tests/test_gpu_hgt_hyper.py tests/test_gpu_dhn.py -x -q > $O/pytest_prog.log 2>&1; echo "exit $?" >> $O/pytest_prog.log
for c in arxiv mag hyper; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_arxiv.csv \
  python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --eager > $O/ncu_launch_arxiv.log 2>&1
