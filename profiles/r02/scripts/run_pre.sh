# neighbour-metadata prefetch in the C3 / C4 walks, fixed-order parallel column-sum finals:
# DHN + epilogue/projection parity, benches, compute-sanitizer on the tiny tier
set -u
O=gpurun_out/r02_pre; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x --durations=5 > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_programs.py tests/test_gpu_train.py -q -x > $O/pytest_parity.log 2>&1; echo "exit $?" >> $O/pytest_parity.log
timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01.json 2> $O/dhn01.err
timeout 900 python bench.py --config arxiv --no-cpu-baseline > $O/bench_arxiv.json 2> $O/bench_arxiv.err
timeout 1500 python bench.py --config dhn --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_dhn.json 2> $O/bench_dhn.err
for part in lja proj; do
  SANITIZE_PART=$part timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/racecheck_$part.log 2>&1; echo "exit $?" >> $O/racecheck_$part.log
done
for k in 3 4; do
  SANITIZE_PART=dhn SANITIZE_DHN_N=40 SANITIZE_DHN_K=$k timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/racecheck_dhn_k$k.log 2>&1; echo "exit $?" >> $O/racecheck_dhn_k$k.log
done
CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/memcheck.log 2>&1; echo "exit $?" >> $O/memcheck.log
SANITIZE_PART=dhn SANITIZE_DHN_N=60 timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/synccheck_dhn.log 2>&1; echo "exit $?" >> $O/synccheck_dhn.log
timeout 900 python bench.py --config arxiv --l2-window --no-cpu-baseline --no-e2e > $O/bench_arxiv_l2w.json 2> $O/bench_arxiv_l2w.err
timeout 900 ncu --set full --clock-control none -k regex:'lean_kernel' -c 6 -o $O/prof_arxiv_l2w -f \
  python bench.py --config arxiv --l2-window --steps 1 --warmup 1 --seeds 42 --no-e2e --no-cpu-baseline > $O/ncu_l2w.log 2>&1
ncu -i $O/prof_arxiv_l2w.ncu-rep --page raw --csv > $O/prof_arxiv_l2w_raw.csv 2>&1
rm -f $O/prof_arxiv_l2w.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'dhn4s_kernel' -c 1 -o $O/prof_dhn4s -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn4s.log 2>&1
ncu -i $O/prof_dhn4s.ncu-rep --page raw --csv > $O/prof_dhn4s_raw.csv 2>&1
rm -f $O/prof_dhn4s.ncu-rep
