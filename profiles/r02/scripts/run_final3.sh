# round-2 final evidence (second pass, end of round): smoke, full GPU suite, bench lines for
# every config and the reference arm, ncu launch lists and full captures
set -u
O=gpurun_out/r02_final3; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt; lscpu >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
for c in arxiv hyper cora; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 2400 python bench.py --config dhn --steps 2 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_mag.json 2> $O/bench_ref_mag.err
for c in mag arxiv hyper; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --seeds 42 \
    --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'st_kernel|sm_d_kernel|tc_gemm|tc_projt' -c 24 -o /tmp/ncu/prof_mag -f \
  python bench.py --config mag --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_mag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lean_kernel|epi_bwd|tc_gemm|tc_projt|splitk|colsum' -c 28 -o /tmp/ncu/prof_arxiv -f \
  python bench.py --config arxiv --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_arxiv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lean_kernel' -c 4 -o /tmp/ncu/prof_hyper -f \
  python bench.py --config hyper --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_hyper.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'dhn3_kernel|dhn4s_kernel' -c 3 -o /tmp/ncu/prof_dhn -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_full_dhn.log 2>&1
for c in mag arxiv hyper dhn; do
  ncu -i /tmp/ncu/prof_$c.ncu-rep --page raw --csv > $O/prof_${c}_raw.csv 2>&1
done
ncu -i /tmp/ncu/prof_mag.ncu-rep --page source --csv > $O/prof_mag_source.csv 2>&1
