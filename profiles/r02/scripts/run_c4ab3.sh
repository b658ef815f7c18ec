# C4: partition probe off (new default) vs the full table for every root, two repeats each
set -u
O=gpurun_out/r02_c4ab3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { timeout 600 python bench.py --config dhn --dhn-scale 0.1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/dhn01_$1.json 2> $O/dhn01_$1.err; }
run default_a
RNN_DHN_FULL_TABLE=1 run fulltable_a
run default_b
RNN_DHN_FULL_TABLE=1 run fulltable_b
RNN_DHN_PROBE=1 run probe
timeout 900 python -m pytest tests/test_gpu_dhn_scale.py -q -x -k "partitioned or overflow or exact or c3" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
