# fused ReLU projection backward, BF16 projections, L2 persisting window experiment
set -u
O=gpurun_out/r02c; mkdir -p $O /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -k "relu or bf16 or projection" tests/test_gpu_programs.py tests/test_gpu_train.py -q -x --durations=8 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python bench.py --config arxiv --seeds 42,43 --no-cpu-baseline --no-e2e > $O/arxiv.json 2> $O/arxiv.err
timeout 600 python bench.py --config cora --seeds 42 --no-cpu-baseline --no-e2e > $O/cora.json 2> $O/cora.err
timeout 600 python bench.py --config arxiv --seeds 42 --eager --no-cpu-baseline --no-e2e > $O/arxiv_eager.json 2> $O/arxiv_eager.err
timeout 600 python bench.py --config arxiv --seeds 42 --l2-window --no-cpu-baseline --no-e2e > $O/arxiv_l2w.json 2> $O/arxiv_l2w.err
timeout 600 python bench.py --config arxiv --seeds 42 --prec bf16 --no-cpu-baseline --no-e2e > $O/arxiv_bf16.json 2> $O/arxiv_bf16.err
for w in off on; do
  extra=""; [ $w = on ] && extra="--l2-window"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --cache-control none --clock-control none -k regex:'lean_kernel|bwd' --csv --log-file $O/ncu_l2w_$w.csv \
    python bench.py --config arxiv --steps 1 --warmup 2 --seeds 42 --eager $extra --no-e2e --no-cpu-baseline > $O/ncu_l2w_$w.log 2>&1
done
