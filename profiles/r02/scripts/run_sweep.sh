O=gpurun_out/r02_sweep; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for ch in 256 1024 4096 16384 100000000; do
  echo "chunk $ch $(RNN_GEMM_CHUNK=$ch timeout 300 python profiles/r02/scripts/sweep_chunk.py 2>&1 | tail -1)" >> $O/chunk.txt
done
echo "chunk 1024 nbuf1 $(RNN_GEMM_NBUF1=1 timeout 300 python profiles/r02/scripts/sweep_chunk.py 2>&1 | tail -1)" >> $O/chunk.txt
for v in "6,4" "8,0" "8,3" "4,4"; do
  RNN_LEAN_EPI_VAR=$v timeout 600 python bench.py --config arxiv --seeds 42 --steps 10 --no-cpu-baseline --no-e2e > $O/arxiv_$v.json 2>/dev/null
done
