# final HEAD: full GPU suite + smoke + default bench line
set -u
O=gpurun_out/r02_head_final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
timeout 2700 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 1500 python bench.py > $O/bench_mag.json 2> $O/bench_mag.err
