O=gpurun_out/r02_san; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python profiles/r02/scripts/sanitize_tiny.py > $O/plain.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python profiles/r02/scripts/sanitize_tiny.py > $O/$tool.log 2>&1
  echo "exit $?" >> $O/$tool.log
done
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
