# ncu evidence refresh at HEAD for the three bandwidth configs (launch lists + full captures)
set -u
O=gpurun_out; mkdir -p $O /tmp/ncu
for c in arxiv hyper mag; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 \
    --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lean_kernel|tc_gemm|tc_projt|splitk' -c 18 -o /tmp/ncu/prof_arxiv -f \
  python bench.py --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_arxiv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'lean_kernel' -c 4 -o /tmp/ncu/prof_hyper -f \
  python bench.py --config hyper --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_hyper.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'st_kernel|sm_d_kernel' -c 16 -o /tmp/ncu/prof_mag -f \
  python bench.py --config mag --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_mag.log 2>&1
for c in arxiv hyper mag; do
  ncu -i /tmp/ncu/prof_$c.ncu-rep --page raw --csv > $O/prof_${c}_raw.csv 2>&1
done
