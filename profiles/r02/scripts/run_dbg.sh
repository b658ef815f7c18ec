O=gpurun_out/r02_dbg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python profiles/r02/scripts/dbg_hgt.py 0.004 > $O/small.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python profiles/r02/scripts/dbg_hgt.py 0.004 > $O/small_memcheck.log 2>&1
timeout 300 python profiles/r02/scripts/dbg_hgt.py 1.0 > $O/full.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dhn_scale.py -q -x --durations=10 > $O/pytest_dhn_scale.log 2>&1
