O=gpurun_out/r02_dbg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python profiles/r02/scripts/dbg_ovf.py > $O/ovf.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python profiles/r02/scripts/dbg_hgt.py 1.0 > $O/full_blocking.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python profiles/r02/scripts/dbg_hgt.py 0.2 > $O/mid_memcheck.log 2>&1
