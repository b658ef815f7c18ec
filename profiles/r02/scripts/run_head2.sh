# round-2 re-entry: evidence at HEAD 5a7fe02 -- smoke, full GPU suite, bench lines, DHN full scale,
# launch lists, ncu captures of the two kernels furthest below their roofline (dhn4, proj bwd)
set -u
O=gpurun_out/r02_head2; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
for c in arxiv hyper cora; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 2400 python bench.py --config dhn --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_dhn.json 2> $O/bench_dhn.err
timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_dhn01.json 2> $O/bench_dhn01.err
for c in mag arxiv; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --seeds 42 \
    --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'tc_gemm|tc_projt|splitk' -c 12 -o /tmp/ncu/prof_mag_proj -f \
  python bench.py --config mag --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_mag.log 2>&1
ncu -i /tmp/ncu/prof_mag_proj.ncu-rep --page raw --csv > $O/prof_mag_proj_raw.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dhn4_kernel -c 2 -o /tmp/ncu/dhn4 -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn4.log 2>&1
ncu -i /tmp/ncu/dhn4.ncu-rep --page raw --csv > $O/dhn4_raw.csv 2>&1
ncu -i /tmp/ncu/dhn4.ncu-rep --page source --csv > $O/dhn4_source.csv 2>&1
cp /tmp/ncu/dhn4.ncu-rep /tmp/ncu/prof_mag_proj.ncu-rep $O/ 2>/dev/null
