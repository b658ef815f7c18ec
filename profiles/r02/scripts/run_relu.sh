set -u
O=gpurun_out/r02_relu; mkdir -p $O
timeout 300 python profiles/r02/scripts/probe_relu.py > $O/probe.log 2>&1
PROBE_ONE=relu timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_projt -c 8 -o $O/relu -f python profiles/r02/scripts/probe_relu.py > $O/ncu.log 2>&1
ncu -i $O/relu.ncu-rep --page raw --csv > $O/relu_raw.csv 2>&1
ncu -i $O/relu.ncu-rep --page source --csv > $O/relu_source.csv 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "bf16" > $O/pytest_bf16.log 2>&1; echo "exit $?" >> $O/pytest_bf16.log
