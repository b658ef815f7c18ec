set -u
O=gpurun_out/r02_head; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi > $O/nvsmi.txt 2>&1; nproc > $O/nproc.txt; lscpu >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py --config mag --steps 10 --warmup 3 > $O/bench_mag.json 2> $O/bench_mag.err
timeout 600 python bench.py > $O/bench_arxiv.json 2> $O/bench_arxiv.err
