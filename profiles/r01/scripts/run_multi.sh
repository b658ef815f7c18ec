# N > 1 bench path on a 1-GPU box: 2 ranks sharing cuda:0 over gloo (functional check only)
set -u
O=gpurun_out; mkdir -p $O
for c in arxiv hyper mag; do
  RNN_BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config $c --steps 3 --warmup 3 \
    --no-cpu-baseline --no-e2e > $O/bench_multi_$c.json 2> $O/bench_multi_$c.err
  echo "exit $?" >> $O/bench_multi_$c.err
done
