# C4 slot walk A/B at 0.1 scale: neighbour prefetch, partition probe, per-root table size
set -u
O=gpurun_out/r02_c4ab; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/dhn01_$1.json 2> $O/dhn01_$1.err; }
run default
RNN_DHN_NO_PREFETCH=1 run noprefetch
RNN_DHN_NO_PROBE=1 run noprobe
RNN_DHN_FULL_TABLE=1 run fulltable
RNN_DHN_NO_PREFETCH=1 RNN_DHN_FULL_TABLE=1 run neither
timeout 900 python -m pytest tests/test_gpu_dhn_scale.py -q -x -k "partitioned or overflow or exact" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
