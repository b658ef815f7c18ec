# slot-indexed C4 walk + two-chunk C3 walk: DHN parity, 0.1-scale A/B, full scale, ncu
set -u
O=gpurun_out/r02_c4s; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x --durations=8 > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_slot.json 2> $O/dhn01_slot.err
RNN_DHN_COMPACT_IDS=1 timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_compact.json 2> $O/dhn01_compact.err
for pk in 2048 4096; do
  RNN_DHN_PART_KEYS=$pk timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01_pk$pk.json 2> $O/dhn01_pk$pk.err
done
timeout 1200 python bench.py --config dhn --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn1_slot.json 2> $O/dhn1_slot.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'dhn4s_kernel|dhn3_kernel' -c 3 -o /tmp/ncu/dhn4s -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_dhn4s.log 2>&1
ncu -i /tmp/ncu/dhn4s.ncu-rep --page raw --csv > $O/dhn4s_raw.csv 2>&1
ncu -i /tmp/ncu/dhn4s.ncu-rep --page source --csv > $O/dhn4s_source.csv 2>&1
