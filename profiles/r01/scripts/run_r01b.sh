set -u
O=gpurun_out; mkdir -p $O /tmp/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_programs.py tests/test_gpu_hgt_hyper.py -x -q > $O/pytest_sub.log 2>&1; echo "exit $?" >> $O/pytest_sub.log
for c in arxiv cora hyper mag; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config arxiv --steps 10 --warmup 3 --no-cpu-baseline --eager > $O/bench_arxiv_eager.json 2> $O/bench_arxiv_eager.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'st_kernel' -s 28 -c 6 -o /tmp/ncu/prof_magbwd -f \
    python bench.py --config mag --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --eager > $O/ncu_full_magbwd.log 2>&1
ncu -i /tmp/ncu/prof_magbwd.ncu-rep --page raw --csv > $O/prof_magbwd_raw.csv 2>&1
timeout 600 ncu --set full --clock-control none -k regex:'tc_|splitk' -s 10 -c 8 -o /tmp/ncu/prof_gemm -f \
    python bench.py --config arxiv --steps 1 --warmup 2 --no-e2e --no-cpu-baseline --eager > $O/ncu_full_gemm.log 2>&1
ncu -i /tmp/ncu/prof_gemm.ncu-rep --page raw --csv > $O/prof_gemm_raw.csv 2>&1
du -sh $O
