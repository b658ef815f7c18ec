O=gpurun_out/r02_dhn; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x --durations=5 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for v in smem l2; do
  if [ $v = l2 ]; then export RNN_DHN_L2SLAB=1; else unset RNN_DHN_L2SLAB; fi
  timeout 900 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_$v.json 2> $O/dhn01_$v.err
done
unset RNN_DHN_L2SLAB
timeout 1500 python bench.py --config dhn --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn1.json 2> $O/dhn1.err
timeout 600 python bench.py --config arxiv --seeds 42 --steps 10 --no-cpu-baseline --no-e2e > $O/arxiv.json 2> $O/arxiv.err
timeout 900 ncu --set full --import-source on --kernel-name regex:dhn4_kernel --launch-count 1 -o $O/dhn4_smem python bench.py --config dhn --dhn-scale 0.1 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn4.log 2>&1
ncu -i $O/dhn4_smem.ncu-rep --page raw --csv > $O/dhn4_smem_raw.csv 2>&1
for part in index lja train dhn proj; do
  SANITIZE_PART=$part timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/racecheck_$part.log 2>&1
  echo "exit $?" >> $O/racecheck_$part.log
done
CUDA_MODULE_LOADING=EAGER timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/memcheck_eager.log 2>&1
echo "exit $?" >> $O/memcheck_eager.log
