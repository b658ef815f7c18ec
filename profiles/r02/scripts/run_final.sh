# round-2 final evidence at HEAD: full GPU suite, smoke, bench lines, ncu launch lists + captures
set -u
O=gpurun_out/r02_final; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=25 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
for c in arxiv hyper cora; do
  timeout 1200 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 1800 python bench.py --config dhn --steps 3 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
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
  -k regex:'lean_kernel|epi_bwd|tc_gemm|tc_projt|splitk' -c 24 -o /tmp/ncu/prof_arxiv -f \
  python bench.py --config arxiv --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_arxiv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lean_kernel' -c 4 -o /tmp/ncu/prof_hyper -f \
  python bench.py --config hyper --steps 1 --warmup 1 --seeds 42 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_hyper.log 2>&1
for c in mag arxiv hyper; do
  ncu -i /tmp/ncu/prof_$c.ncu-rep --page raw --csv > $O/prof_${c}_raw.csv 2>&1
done
cp /tmp/ncu/prof_mag.ncu-rep $O/ 2>/dev/null
# DHN C3 / C4 (L2-slab default) full captures, 0.03-scale products graph (the 0.1-scale C4 replay timed out in ncu)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dhn4_kernel -c 1 -o /tmp/ncu/dhn4_l2 -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn4.log 2>&1
ncu -i /tmp/ncu/dhn4_l2.ncu-rep --page raw --csv > $O/dhn4_l2_raw.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dhn3_kernel -c 1 -o /tmp/ncu/dhn3 -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn3.log 2>&1
ncu -i /tmp/ncu/dhn3.ncu-rep --page raw --csv > $O/dhn3_raw.csv 2>&1
# sanitizers: first-launch report probe, DHN racecheck per k on a 40-node graph
SANITIZE_FIRST=gather CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/memcheck_first_gather.log 2>&1; echo "exit $?" >> $O/memcheck_first_gather.log
for k in 2 3 4; do
  SANITIZE_PART=dhn SANITIZE_DHN_N=40 SANITIZE_DHN_K=$k timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/racecheck_dhn_k$k.log 2>&1; echo "exit $?" >> $O/racecheck_dhn_k$k.log
done
