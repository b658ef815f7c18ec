O=gpurun_out/r02_dbg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python profiles/r02/scripts/dbg_dw.py > $O/dw.log 2>&1
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x > $O/shard.log 2>&1
