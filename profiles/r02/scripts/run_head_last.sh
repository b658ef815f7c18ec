# HEAD at the end of round 2: full GPU suite + smoke, DHN ncu capture of the final walk code
set -u
O=gpurun_out/r02_head_last; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'dhn3_kernel|dhn4s_kernel' -c 3 -o /tmp/ncu/prof_dhn -f \
  python bench.py --config dhn --dhn-scale 0.03 --steps 1 --warmup 0 --seeds 42 --no-cpu-baseline --no-e2e --eager > $O/ncu_full_dhn.log 2>&1
ncu -i /tmp/ncu/prof_dhn.ncu-rep --page raw --csv > $O/prof_dhn_raw.csv 2>&1
