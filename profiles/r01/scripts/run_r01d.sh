set -u
O=gpurun_out; mkdir -p $O /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py -k "projection" -x -q > $O/pytest_proj.log 2>&1; echo "exit $?" >> $O/pytest_proj.log
timeout 600 python bench.py --config arxiv --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_arxiv.json 2> $O/bench_arxiv.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'tc_projt|tc_gemm' -s 6 -c 3 -o /tmp/ncu/prof_projt -f \
  python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --eager > $O/ncu_projt.log 2>&1
ncu -i /tmp/ncu/prof_projt.ncu-rep --page raw --csv > $O/prof_projt_raw.csv 2>&1
ncu -i /tmp/ncu/prof_projt.ncu-rep --page source --csv --kernel-name regex:tc_projt --launch-skip 0 --launch-count 1 > $O/prof_projt_source.csv 2>&1
ncu -i /tmp/ncu/prof_projt.ncu-rep --page details --csv > $O/prof_projt_details.csv 2>&1
