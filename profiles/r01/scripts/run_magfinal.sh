set -u
O=gpurun_out; mkdir -p $O /tmp/ncu
timeout 900 python bench.py --config mag --steps 10 --warmup 3 > $O/bench_mag.json 2> $O/bench_mag.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_mag.csv python bench.py --config mag --steps 1 --warmup 3 \
  --no-e2e --no-cpu-baseline > $O/ncu_launch_mag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'st_kernel|sm_d_kernel' -c 16 -o /tmp/ncu/prof_mag -f \
  python bench.py --config mag --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_mag.log 2>&1
ncu -i /tmp/ncu/prof_mag.ncu-rep --page raw --csv > $O/prof_mag_raw.csv 2>&1
