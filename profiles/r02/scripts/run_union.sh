# deterministic load-balanced C3 at 4 x 256, C4 4 hits in flight; HGT union fused into the
# softmax store + accumulating dQ: tests, MAG / DHN benches
set -u
O=gpurun_out/r02_union; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "union or softmax" > $O/pytest_union.log 2>&1; echo "exit $?" >> $O/pytest_union.log
timeout 900 python -m pytest tests/test_gpu_hgt_hyper.py tests/test_gpu_attention_variants.py tests/test_gpu_shard.py -q -x > $O/pytest_hgt.log 2>&1; echo "exit $?" >> $O/pytest_hgt.log
timeout 1500 python -m pytest tests/test_gpu_dhn.py tests/test_gpu_dhn_scale.py -q -x --durations=5 > $O/pytest_dhn.log 2>&1; echo "exit $?" >> $O/pytest_dhn.log
timeout 1200 python bench.py --no-cpu-baseline > $O/bench_mag.json 2> $O/bench_mag.err
timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn01.json 2> $O/dhn01.err
timeout 1200 python bench.py --config dhn --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/dhn1.json 2> $O/dhn1.err
timeout 900 python -m pytest tests/test_gpu_full_scale.py -q -x -k mag > $O/pytest_mag_full.log 2>&1; echo "exit $?" >> $O/pytest_mag_full.log
