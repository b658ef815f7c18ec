# pass B (group-major dQ gather) rows in flight x resident CTAs around (2, 6)
set -u
O=gpurun_out/r02_stvar3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in 4,3,1,4,2,6 4,3,1,4,2,8 4,3,1,4,3,6 4,3,1,4,1,6 4,3,1,4,1,8 4,3,1,4,2,5 4,3,1,4,4,4; do
  RNN_ST_VAR=$v timeout 600 python bench.py --seeds 42 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/mag_$v.json 2> $O/mag_$v.err
done
