#!/usr/bin/env bash
# Final round-1 evidence at HEAD (run under gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash profiles/run_r01f.sh [tests|bench|ncu|all]'
# Numbers printed by the ncu passes are never bench values (B200_PROFILING.md).
set -u
O=gpurun_out
mkdir -p $O /tmp/ncu
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1

if [[ $what == tests || $what == all ]]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
fi

if [[ $what == bench || $what == all ]]; then
  timeout 600 python bench.py > $O/bench_arxiv.json 2> $O/bench_arxiv.err
  for c in cora hyper mag; do
    timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
  done
  timeout 900 python bench.py --config dhn --steps 3 --warmup 3 > $O/bench_dhn.json 2> $O/bench_dhn.err
  timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
fi

if [[ $what == ncu || $what == all ]]; then
  for c in arxiv hyper mag dhn; do
    # launch list of the whole process (index build + warm-up + 1 step): kernel SHARE
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 \
      --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1
  done
  # full captures of one eager step's hot kernels (first launches after the index build)
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'lean_kernel|tc_gemm|tc_projt|splitk' -c 18 -o /tmp/ncu/prof_arxiv -f \
    python bench.py --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_arxiv.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'st_kernel' -c 12 -o /tmp/ncu/prof_mag -f \
    python bench.py --config mag --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_mag.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'lean_kernel' -c 4 -o /tmp/ncu/prof_hyper -f \
    python bench.py --config hyper --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_hyper.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'dhn[34]_kernel' -c 2 -o /tmp/ncu/prof_dhn -f \
    python bench.py --config dhn --steps 1 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu_full_dhn.log 2>&1
  for c in arxiv mag hyper dhn; do
    if [[ -f /tmp/ncu/prof_$c.ncu-rep ]]; then
      ncu -i /tmp/ncu/prof_$c.ncu-rep --page raw --csv > $O/prof_${c}_raw.csv 2>&1
    fi
  done
  ls -la /tmp/ncu > $O/ncu_reps.txt
fi
du -sh $O
echo done
