O=gpurun_out/r02_dbg; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python profiles/r02/scripts/dbg_prec.py > $O/prec.log 2>&1
